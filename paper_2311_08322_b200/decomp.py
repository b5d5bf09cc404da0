"""Horizontal domain decomposition and halo exchange.

The reference has no multi-process path (stencilforge ``SPEC.md:12``; its
only parallelism is OpenMP inside one generated kernel, ``gen.py:331-360``).
This module adds the B200-side one: a 2-D (i, j) split of the compute domain
over the ranks of one node, one process per GPU, k never split (FORWARD /
BACKWARD recurrences run along k).

* ``Decomposition`` -- the rank grid (1x1, 2x1, 2x2, 4x2, ...), each rank's
  sub-domain in global coordinates and its face neighbours (non-periodic).
* ``HaloExchanger`` -- refreshes the halo of a field of extent (hi, hj) from
  the neighbours: i-faces first (full storage width), then j-faces over the
  full i range including the freshly received i-halos, so corners arrive
  without diagonal messages.  Transport is ``torch.distributed`` point-to-
  point (``batch_isend_irecv``): NCCL over NVLink for device fields (faces
  packed / unpacked by ``gts_b200_pack_box`` / ``gts_b200_unpack_box``
  kernels on the exchange stream), gloo for host arrays (used by the CPU
  tests of this logic).
* ``DecomposedStep`` -- runs a stencil on the interior (which needs no halo)
  while the exchange is in flight, then ONE frame launch over the tiles
  touching the halo-dependent band (``split_launches``; the four boundary
  strips for stencils without a frame launch); every point is computed by
  exactly the same instructions as in an undecomposed run, so the result is
  bitwise identical.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

GRIDS = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2), 16: (4, 4)}


def choose_grid(world: int) -> tuple:
    if world in GRIDS:
        return GRIDS[world]
    pi = int(np.sqrt(world))
    while world % pi:
        pi -= 1
    return (world // pi, pi)


def _split(n: int, parts: int, idx: int) -> tuple:
    base, rem = divmod(n, parts)
    lo = idx * base + min(idx, rem)
    return lo, lo + base + (1 if idx < rem else 0)


@dataclass
class Decomposition:
    global_domain: tuple  # (ni, nj, nk)
    grid: tuple  # (pi, pj)
    rank: int

    def __post_init__(self):
        pi, pj = self.grid
        if not 0 <= self.rank < pi * pj:
            raise ValueError(f"rank {self.rank} outside the {pi}x{pj} grid")
        self.ri, self.rj = divmod(self.rank, pj)
        ni, nj, nk = self.global_domain
        self.i0, self.i1 = _split(ni, pi, self.ri)
        self.j0, self.j1 = _split(nj, pj, self.rj)
        if self.i1 <= self.i0 or self.j1 <= self.j0:
            raise ValueError(f"grid {self.grid} too fine for domain {self.global_domain}")

    @property
    def local_domain(self) -> tuple:
        return (self.i1 - self.i0, self.j1 - self.j0, self.global_domain[2])

    def neighbour(self, di: int, dj: int) -> Optional[int]:
        pi, pj = self.grid
        ri, rj = self.ri + di, self.rj + dj
        if 0 <= ri < pi and 0 <= rj < pj:
            return ri * pj + rj
        return None

    def scatter(self, global_storage_array: np.ndarray, halo: tuple) -> np.ndarray:
        """This rank's storage box (local domain + halo) of a global logical
        array laid out with the same halo (global storage coordinates)."""
        hi, hj = halo
        # always a copy: a slice of full trailing extent is already contiguous,
        # and ascontiguousarray would hand back a view aliasing the global array
        return np.array(
            global_storage_array[self.i0: self.i1 + 2 * hi, self.j0: self.j1 + 2 * hj, :], copy=True)


class _HostOps:
    """Face pack / unpack / buffers on host numpy arrays (gloo transport)."""

    def __init__(self, torch):
        self.torch = torch

    def alloc(self, count, dtype):
        return self.torch.empty(count, dtype=dtype)

    def pack(self, buf, field, box):
        (i0, j0, k0), (n_i, n_j, n_k) = box
        v = field[i0: i0 + n_i, j0: j0 + n_j, k0: k0 + n_k]
        buf.copy_(self.torch.from_numpy(np.ascontiguousarray(v.transpose(2, 0, 1))).reshape(-1))

    def unpack(self, field, buf, box):
        (i0, j0, k0), (n_i, n_j, n_k) = box
        arr = buf.numpy().reshape(n_k, n_i, n_j).transpose(1, 2, 0)
        field[i0: i0 + n_i, j0: j0 + n_j, k0: k0 + n_k] = arr

    def synchronize(self):
        pass


class _DeviceOps:
    """Face pack / unpack kernels of libgts_b200.so on the exchange stream;
    buffers are torch CUDA tensors so NCCL can move them."""

    def __init__(self, torch, stream: int):
        from . import native

        self.torch, self.native, self.stream = torch, native, stream

    def alloc(self, count, dtype):
        return self.torch.empty(count, dtype=dtype, device="cuda")

    def _args(self, st, box):
        (i0, j0, k0), (n_i, n_j, n_k) = box
        return [st.base_address(), *st.strides, i0, j0, k0, n_i, n_j, n_k, st.itemsize, self.stream]

    def pack(self, buf, st, box):
        a = self._args(st, box)
        self.native.call("gts_b200_pack_box", buf.data_ptr(), *a)

    def unpack(self, st, buf, box):
        a = self._args(st, box)
        self.native.call("gts_b200_unpack_box", a[0], buf.data_ptr(), *a[1:])

    def synchronize(self):
        self.native.synchronize(self.stream)


class HaloExchanger:
    """Halo refresh of one field (storage = local domain + (hi, hj) halo)."""

    def __init__(self, decomp: Decomposition, halo: tuple, dtype: str, device: bool = True,
                 stream: Optional[int] = None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.decomp, self.halo = decomp, tuple(halo)
        self.tdtype = torch.float32 if dtype == "f32" else torch.float64
        if device:
            from . import native

            self.ops = _DeviceOps(torch, stream if stream is not None else native.default_stream())
        else:
            self.ops = _HostOps(torch)
        self.device = device
        ni, nj, nk = decomp.local_domain
        hi, hj = self.halo
        self._bufs = {}
        for key, count in (("i", hi * (nj + 2 * hj) * nk), ("j", (ni + 2 * hi) * hj * nk)):
            if count:
                self._bufs[key] = [self.ops.alloc(count, self.tdtype) for _ in range(4)]

    def _phase(self, field, axis: str):
        """Exchange the two faces along one axis: returns the list of p2p ops."""
        ni, nj, nk = self.decomp.local_domain
        hi, hj = self.halo
        if axis == "i":
            if hi == 0:
                return []
            # full storage width: a rank on the global j boundary must also
            # receive the neighbour's copy of the global j-halo columns; j-halo
            # columns owned by a j-neighbour are overwritten in phase 2
            lo_n, hi_n = self.decomp.neighbour(-1, 0), self.decomp.neighbour(1, 0)
            span = (hi, nj + 2 * hj, nk)
            send_lo, recv_lo = ((hi, 0, 0), span), ((0, 0, 0), span)
            send_hi, recv_hi = ((ni, 0, 0), span), ((ni + hi, 0, 0), span)
        else:
            if hj == 0:
                return []
            lo_n, hi_n = self.decomp.neighbour(0, -1), self.decomp.neighbour(0, 1)
            span = (ni + 2 * hi, hj, nk)
            send_lo, recv_lo = ((0, hj, 0), span), ((0, 0, 0), span)
            send_hi, recv_hi = ((0, nj, 0), span), ((0, nj + hj, 0), span)
        sb_lo, rb_lo, sb_hi, rb_hi = self._bufs[axis]
        ops, unpacks = [], []
        P2P = self.dist.P2POp
        if lo_n is not None:
            self.ops.pack(sb_lo, field, send_lo)
            ops += [P2P(self.dist.isend, sb_lo, lo_n), P2P(self.dist.irecv, rb_lo, lo_n)]
            unpacks.append((rb_lo, recv_lo))
        if hi_n is not None:
            self.ops.pack(sb_hi, field, send_hi)
            ops += [P2P(self.dist.isend, sb_hi, hi_n), P2P(self.dist.irecv, rb_hi, hi_n)]
            unpacks.append((rb_hi, recv_hi))
        return ops, unpacks

    def exchange_async(self, field) -> None:
        """Device mode, no host synchronisation: pack, NCCL send/recv and
        unpack are all enqueued on the exchanger's stream, which must be the
        torch current stream (NCCL orders its kernels on it)."""
        assert self.device
        for axis in ("i", "j"):
            res = self._phase(field, axis)
            if not res:
                continue
            ops, unpacks = res
            if ops:
                for req in self.dist.batch_isend_irecv(ops):
                    req.wait()  # stream-ordered for NCCL; no host block
            for buf, box in unpacks:
                self.ops.unpack(field, buf, box)

    def exchange(self, field) -> None:
        """Blocking-on-stream halo refresh of ``field`` (a DeviceFieldStorage
        in device mode, a logical numpy array in host mode)."""
        for axis in ("i", "j"):
            res = self._phase(field, axis)
            if not res:
                continue
            ops, unpacks = res
            if ops:
                if self.device:
                    self.ops.synchronize()  # packed faces complete before NCCL reads them
                for req in self.dist.batch_isend_irecv(ops):
                    req.wait()
                if self.device:
                    self.torch.cuda.current_stream().synchronize()
            for buf, box in unpacks:
                self.ops.unpack(field, buf, box)
        if self.device:
            self.ops.synchronize()


def strips(domain: tuple, halo: tuple) -> list:
    """Interior + boundary strips of a local domain for overlap: the interior
    [hi, ni-hi) x [hj, nj-hj) reads no halo cell of a field of extent
    (hi, hj); the four strips cover the rest exactly once."""
    ni, nj, nk = domain
    hi, hj = halo
    out = []
    if ni > 2 * hi and nj > 2 * hj:
        out.append(("interior", (hi, hj), (ni - 2 * hi, nj - 2 * hj)))
        out.append(("north", (0, 0), (hi, nj)))
        out.append(("south", (ni - hi, 0), (hi, nj)))
        out.append(("west", (hi, 0), (ni - 2 * hi, hj)))
        out.append(("east", (hi, nj - hj), (ni - 2 * hi, hj)))
    else:
        out.append(("all", (0, 0), (ni, nj)))
    return [(name, o, (s[0], s[1], nk)) for name, o, s in out if s[0] > 0 and s[1] > 0]


def call_on_strip(stencil, fields: dict, scalars: dict, offset: tuple, size: tuple) -> None:
    """Run a compiled stencil on a sub-rectangle of the local domain: the
    reference's explicit ``origin=`` / ``domain=`` arguments
    (``runtime.py:122-200``), shifted per field."""
    origins = {n: (st.origin[0] + offset[0], st.origin[1] + offset[1], st.origin[2])
               for n, st in fields.items()}
    stencil(domain=tuple(size), origin=origins, **fields, **scalars)


def frame_interior(domain: tuple, band, tile):
    """Offset and size of the interior launch that complements a frame
    launch.  ``band`` = (hi, hj), or per side (ilo, ihi, jlo, jhi) with 0 for
    a side that needs none (no neighbour there).  The frame kernel runs every
    FTI x FTJ tile outside the inner tile rectangle [ceil(ilo/FTI),
    floor((ni-ihi)/FTI)) x [ceil(jlo/FTJ), floor((nj-jhi)/FTJ)) -- a side
    without a band reaches the last (partial) tile -- (codegen_parallel frame
    variant, ``gts_frame_tile``), so the interior is that rectangle in points,
    clipped to the domain; None when it is empty.  ``tile`` None (a module
    without the query): the halo-free interior, computed twice where frame
    tiles overlap it."""
    from .backend import frame_bands

    ni, nj, nk = domain
    ilo, ihi, jlo, jhi = frame_bands(band)
    if tile is None:
        i0, i1, j0, j1 = ilo, ni - ihi, jlo, nj - jhi
        return ((i0, j0), (i1 - i0, j1 - j0, nk)) if i1 > i0 and j1 > j0 else None
    ti, tj = tile
    fi0, fi1 = -(-ilo // ti), ((ni - ihi) // ti if ihi else -(-ni // ti))
    fj0, fj1 = -(-jlo // tj), ((nj - jhi) // tj if jhi else -(-nj // tj))
    if fi1 <= fi0 or fj1 <= fj0:
        return None
    i0, j0 = fi0 * ti, fj0 * tj
    return (i0, j0), (min(fi1 * ti, ni) - i0, min(fj1 * tj, nj) - j0, nk)


def neighbour_sides(decomposition) -> tuple:
    """(low-i, high-i, low-j, high-j): whether a neighbour lies on that side."""
    return tuple(decomposition.neighbour(di, dj) is not None
                 for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)))


def split_launches(module, domain: tuple, halo: tuple, fields: dict, scalars: dict, stream: int,
                   has_neighbours):
    """(interior launchers, boundary launchers) of one decomposed step.

    ``has_neighbours``: a bool (all four sides or none) or per side (low-i,
    high-i, low-j, high-j; ``neighbour_sides``).  Without neighbours: one
    launch of the whole local domain.  Otherwise an interior box that reads
    no halo cell of a side with a neighbour runs while the halo is in
    flight, and the rest after it lands (a side without a neighbour keeps
    its static boundary halo, so the interior reaches it):

    * ONE frame launch when the module supports it (a single fused PARALLEL
      kernel whose recomputation is idempotent, codegen ``frame_ok``): the
      whole domain, enumerating only the thin tiles that touch the band
      (Module.frame_launcher), with the interior launch on exactly the
      frame's inner tile rectangle (``frame_interior``) -- 2 launches per step;
    * otherwise the interior [hi, ni-hi) x [hj, nj-hj) and the four boundary
      strips (5 launches per step)."""
    sides = (has_neighbours,) * 4 if isinstance(has_neighbours, bool) else tuple(bool(x) for x in has_neighbours)
    if not any(sides):
        return [module.launcher(domain, fields, scalars, stream)], []
    parts = strips(domain, halo)
    if module.frame_supported and any(name == "interior" for name, _, _ in parts):
        # the interior launch covers exactly the frame launch's inner tile
        # rectangle (frame tiles of FTI x FTJ points touching the band are
        # the frame's): every point is computed once
        hi, hj = halo
        band = (hi * sides[0], hi * sides[1], hj * sides[2], hj * sides[3])
        interior = []
        box = frame_interior(domain, band, getattr(module, "frame_tile", None))
        if box is not None:
            (i0, j0), size = box
            interior = [module.launcher(size, fields, scalars, stream, (i0, j0, 0))]
        boundary = [module.frame_launcher(domain, fields, scalars, stream, band)]
        return interior, boundary
    interior = [module.launcher(size, fields, scalars, stream, (off[0], off[1], 0))
                for name, off, size in parts if name in ("interior", "all")]
    boundary = [module.launcher(size, fields, scalars, stream, (off[0], off[1], 0))
                for name, off, size in parts if name not in ("interior", "all")]
    return interior, boundary


def upload_pending(storages, stream: int) -> None:
    """Pending host writes land before a capture: an upload (a synchronous
    copy) cannot be enqueued while the stream is being captured."""
    seen = set()
    for st in storages:
        if id(st) not in seen and hasattr(st, "to_device"):
            seen.add(id(st))
            st.to_device(stream)


class _GraphReplay:
    """``steps`` steps of a decomposed step replayed from one CUDA graph, or
    (``graph=None``: the capture was refused, e.g. by a NCCL build without
    stream-capture support) re-enqueued eagerly step by step."""

    def __init__(self, step, graph, steps: int, written: list):
        self.step, self.graph, self.steps, self.written = step, graph, steps, written

    def launch(self) -> None:
        if self.graph is not None:
            self.graph.launch()
        else:
            for _ in range(self.steps):
                self.step()
        for w in self.written:  # storages written by the replay: host mirrors are stale
            w.mark_device_written(self.step.compute)


class DecomposedStep:
    """One time step of a PARALLEL stencil on a decomposed domain, fully
    asynchronous, in 2 stencil launches: the halo exchange of ``halo_field``
    (pack -> NCCL send/recv -> unpack on the communication stream) overlaps
    the interior launch on the compute stream; the frame launch
    (``split_launches``) runs once the halos have landed.  No host
    synchronisation inside the step, and ``graph(n)`` captures n steps --
    the NCCL calls included -- into one CUDA graph."""

    def __init__(self, stencil, decomposition: Decomposition, fields: dict, scalars: dict,
                 halo_field: str, halo: tuple, split=None):
        """``split``: interior + frame launches even without neighbours (the
        1-GPU measurement of what the split costs): True for all four sides,
        or per side (low-i, high-i, low-j, high-j); default: the sides that
        have a neighbour (``neighbour_sides``)."""
        import torch

        from . import native

        self.torch, self.native = torch, native
        self.compute = self.stream = native.default_stream()
        self.comm = native.aux_stream("nccl-halo")
        self.decomp = decomposition
        self.module = stencil.build_info["module"]
        self.fields = fields
        dom = decomposition.local_domain
        has_nb = any(decomposition.neighbour(di, dj) is not None
                     for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)))
        self.exchanger = None
        if has_nb:
            self.exchanger = HaloExchanger(decomposition, halo, fields[halo_field].dtype, device=True,
                                           stream=self.comm)
            self.field = fields[halo_field]
            self._comm_t = torch.cuda.ExternalStream(self.comm)
        self.interior, self.boundary = split_launches(self.module, dom, halo, fields, scalars, self.compute,
                                                      neighbour_sides(decomposition) if split is None else split)
        self.launches_per_step = len(self.interior) + len(self.boundary)
        self._ev_start, self._ev_halo = native.Event(), native.Event()

    def __call__(self) -> None:
        n = self.native
        if self.exchanger is not None:
            self._ev_start.record_dep(self.compute)  # the field is final for this step
            n.call("gts_b200_stream_wait_event", self.comm, self._ev_start.ptr)
            with self.torch.cuda.stream(self._comm_t):
                self.exchanger.exchange_async(self.field)
            self._ev_halo.record_dep(self.comm)
        for go in self.interior:
            go()
        if self.exchanger is not None:
            n.call("gts_b200_stream_wait_event", self.compute, self._ev_halo.ptr)
        for go in self.boundary:
            go()
        if self.exchanger is not None:
            self.field.mark_device_written(self.compute)  # halo rewritten (joined into compute)

    def graph(self, steps: int) -> _GraphReplay:
        """``steps`` steps captured into one CUDA graph on the compute stream
        (the communication stream joins through the fork / join events; NCCL
        send / recv are stream-capturable).  If the capture is refused the
        replay falls back to eager enqueues."""
        written = [self.fields[name] for name in self.module.written]
        if self.exchanger is not None:
            written.append(self.field)  # its halo is rewritten by the unpack
        upload_pending(self.fields.values(), self.compute)
        g = self.native.Graph(self.compute)
        try:
            with g.capture():
                for _ in range(steps):
                    self()
        except Exception:  # noqa: BLE001 - capture refused: eager replay
            self.native.synchronize(self.compute)
            self.native.synchronize(self.comm)
            return _GraphReplay(self, None, steps, written)
        return _GraphReplay(self, g, steps, written)


# ---------------------------------------------------------------------------
# Peer-memory transport (no NCCL on the data path)
# ---------------------------------------------------------------------------
# direction index d of a face neighbour, and the direction it sees us in
DIRS = ((-1, 0), (1, 0), (0, -1), (0, 1))  # i-lo, i-hi, j-lo, j-hi
OPP = (1, 0, 3, 2)
ARRIVED, ACKED = 0, 4  # flag word = base + d: "halo from d landed (step)", "d consumed my puts (step)"


def face_puts(decomp: Decomposition, halo: tuple, axis: str) -> list:
    """The face copies of one exchange phase, as (direction, src box in my
    storage, dst box origin in the neighbour's storage, box size): my
    boundary rows go straight into the neighbour's halo.  Phase "i" covers the
    interior columns plus the global j-halo columns; phase "j" the full
    storage height including the i-halo rows received in phase "i", so
    corners arrive without diagonal messages.  Unlike HaloExchanger (where
    the receiver unpacks in order) two ranks write into one halo here, so the
    boxes never overlap."""
    ni, nj, nk = decomp.local_domain
    hi, hj = halo
    out = []
    for d in ((0, 1) if axis == "i" else (2, 3)):
        nb = decomp.neighbour(*DIRS[d])
        if nb is None:
            continue
        nd = Decomposition(decomp.global_domain, decomp.grid, nb)
        nni, nnj, _ = nd.local_domain
        if axis == "i":
            if hi == 0:
                continue
            # j-halo columns that a j-neighbour rewrites in phase j are left
            # out: the two writes come from different ranks, unordered, and
            # phase j carries the right (diagonal) values; the global j-halo
            # columns travel here (an i-neighbour shares our j-neighbours)
            c0 = hj if decomp.neighbour(0, -1) is not None else 0
            c1 = nj + hj if decomp.neighbour(0, 1) is not None else nj + 2 * hj
            size = (hi, c1 - c0, nk)
            src = (hi, c0, 0) if d == 0 else (ni, c0, 0)
            dst = (nni + hi, c0, 0) if d == 0 else (0, c0, 0)
        else:
            if hj == 0:
                continue
            size = (ni + 2 * hi, hj, nk)
            src = (0, hj, 0) if d == 2 else (0, nj, 0)
            dst = (0, nnj + hj, 0) if d == 2 else (0, 0, 0)
        out.append((d, nb, src, dst, size))
    return out


class PeerHaloExchanger:
    """Halo refresh of one device field by direct peer-memory puts.

    Every rank shares its field allocation and a 64-byte flag block with its
    face neighbours through CUDA IPC (handles exchanged once over
    ``torch.distributed``).  The flags are counters: ARRIVED[d] counts the
    halo puts received from the neighbour in direction d, ACKED[d] the steps
    that neighbour has finished reading what we put.  Per step, on the
    exchange stream:

    * phase i: for each i-neighbour, wait until it acknowledged the previous
      step (its boundary strips no longer read the halo we are about to
      rewrite), copy our boundary rows straight into its halo (P2P stores over
      NVLink / NVSwitch, ``gts_b200_copy_box``), then add 1 to its ARRIVED
      flag (system-scope release, ``gts_b200_flag_add``); wait for our own
      i-halos;
    * phase j: the same for the j-neighbours over the full height (corners
      travel with the i-halo rows received in phase i); wait for our j-halos.

    ``acknowledge`` (after the boundary strips, on the compute stream) bumps
    each neighbour's ACKED flag.  Each wait bumps a private expected count
    in device memory (``gts_b200_flag_wait_next``), so no launch carries a
    step number: a step needs no host synchronisation, no NCCL call, and can
    be captured once into a CUDA graph and replayed.  The only collective is
    the one-off handle exchange."""

    def __init__(self, decomp: Decomposition, halo: tuple, field, stream: int, group=None):
        import ctypes

        import torch.distributed as dist

        from . import native, storage

        if not isinstance(field, storage.DeviceFieldStorage):
            raise TypeError("PeerHaloExchanger needs a DeviceFieldStorage")
        self.native, self.decomp, self.halo, self.field = native, decomp, tuple(halo), field
        self.stream = stream
        self._flags = storage._DeviceBuffer(64, pinned_host=False)  # shared: ARRIVED[4], ACKED[4]
        self._expect = storage._DeviceBuffer(64, pinned_host=False)  # private expected counts
        native.call("gts_b200_memset", self._flags.dptr, 0, 64, stream)
        native.call("gts_b200_memset", self._expect.dptr, 0, 32, stream)
        # the first ACKED wait must pass at once: expected = -1 (+1 -> 0)
        native.call("gts_b200_memset", self._expect.dptr + 32, 0xFF, 32, stream)
        native.synchronize(stream)

        def handle(ptr):
            h, off = ctypes.create_string_buffer(64), ctypes.c_size_t()
            native.call("gts_b200_ipc_get_handle", ptr, h, ctypes.byref(off))
            return h.raw, off.value

        me = {"field": handle(field.base_address()), "strides": tuple(field.strides),
              "flags": handle(self._flags.dptr)}
        world = dist.get_world_size(group)
        allv = [None] * world
        dist.all_gather_object(allv, me, group=group)
        self._opened = []
        self.peer = {}
        for d in range(4):
            nb = decomp.neighbour(*DIRS[d])
            if nb is None:
                continue
            info = allv[nb]
            fp, gp = ctypes.c_void_p(), ctypes.c_void_p()
            native.call("gts_b200_ipc_open", info["field"][0], ctypes.byref(fp))
            native.call("gts_b200_ipc_open", info["flags"][0], ctypes.byref(gp))
            self._opened += [fp.value, gp.value]
            self.peer[d] = (fp.value + info["field"][1], info["strides"], gp.value + info["flags"][1])
        self.puts = {ax: face_puts(decomp, self.halo, ax) for ax in ("i", "j")}
        dist.barrier(group)  # every rank mapped its peers before anyone signals

    @staticmethod
    def _word(base: int, word: int) -> int:
        return base + 8 * word

    def _wait(self, word: int, stream: int) -> None:
        self.native.call("gts_b200_flag_wait_next", self._word(self._flags.dptr, word),
                         self._word(self._expect.dptr, word), stream)

    def exchange_async(self) -> None:
        """Enqueue one halo refresh on the exchange stream (no host sync)."""
        st, f = self.stream, self.field
        item = f.itemsize
        for axis in ("i", "j"):
            for d, nb, src, dst, size in self.puts[axis]:
                base, strides, pflags = self.peer[d]
                self._wait(ACKED + d, st)
                so = sum(a * b for a, b in zip(src, f.strides))
                do = sum(a * b for a, b in zip(dst, strides))
                self.native.call("gts_b200_copy_box", base + do * item, *strides,
                                 f.base_address() + so * item, *f.strides, *size, item, st)
                self.native.call("gts_b200_flag_add", self._word(pflags, ARRIVED + OPP[d]), st)
            for d, *_ in self.puts[axis]:
                self._wait(ARRIVED + d, st)

    def acknowledge(self, stream: int) -> None:
        """After the step's halo readers on ``stream``: neighbours may rewrite
        our halos for the next step."""
        for d, (base, strides, pflags) in self.peer.items():
            self.native.call("gts_b200_flag_add", self._word(pflags, ACKED + OPP[d]), stream)

    def close(self) -> None:
        for p in self._opened:
            try:
                self.native.call("gts_b200_ipc_close", p)
            except Exception:  # pragma: no cover - teardown
                pass
        self._opened = []


class PeerDecomposedStep:
    """DecomposedStep over the peer-memory transport: the halo exchange
    (PeerHaloExchanger, its own stream) overlaps the interior on the compute
    stream; the boundary strips wait for it through an event; the step ends
    by acknowledging the neighbours.  Native streams and events only."""

    def __init__(self, stencil, decomposition: Decomposition, fields: dict, scalars: dict,
                 halo_field: str, halo: tuple, group=None):
        from . import native

        self.native = native
        self.compute = native.default_stream()
        self.comm = native.aux_stream("peer-halo")
        module = stencil.build_info["module"]
        dom = decomposition.local_domain
        self.exchanger = PeerHaloExchanger(decomposition, halo, fields[halo_field], self.comm, group)
        self.fields = fields
        self.written = sorted(module.written)
        self.interior, self.boundary = split_launches(module, dom, halo, fields, scalars, self.compute,
                                                      neighbour_sides(decomposition) if self.exchanger.peer
                                                      else False)
        self.launches_per_step = len(self.interior) + len(self.boundary)
        self._ev_start, self._ev_halo = native.Event(), native.Event()

    def graph(self, steps: int):
        """``steps`` steps captured once into a CUDA graph on the compute
        stream (the exchange stream joins the capture through the fork / join
        events); replay with ``.launch()``."""
        upload_pending(self.fields.values(), self.compute)
        g = self.native.Graph(self.compute)
        with g.capture():
            for _ in range(steps):
                self()
        written = [self.fields[n] for n in self.written]
        peer = self.exchanger.field

        class _Replay:
            graph = g

            def launch(self_) -> None:
                g.launch()
                for w in written:  # storages written by the replay: host mirrors are stale
                    w.mark_device_written()
                peer.mark_device_written()  # neighbours rewrote its halo

        return _Replay()

    def __call__(self) -> None:
        n = self.native
        if self.exchanger.peer:
            self._ev_start.record_dep(self.compute)  # the field is final for this step
            n.call("gts_b200_stream_wait_event", self.comm, self._ev_start.ptr)
            self.exchanger.exchange_async()
            self._ev_halo.record_dep(self.comm)
        for go in self.interior:
            go()
        if self.exchanger.peer:
            n.call("gts_b200_stream_wait_event", self.compute, self._ev_halo.ptr)
        for go in self.boundary:
            go()
        if self.exchanger.peer:
            self.exchanger.acknowledge(self.compute)
            self.exchanger.field.mark_device_written()  # neighbours rewrote its halo


DIRS8 = [(-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0), (1, 1)]


def mirror_boxes(decomp: Decomposition, halo: tuple) -> list:
    """For each existing neighbour in DIRS8 order: (direction index, rank, box)
    with box = (i0, i1, j0, j1), the cells of our local domain that lie in
    that neighbour's halo (faces: the ``halo``-deep boundary band over the
    full other extent; corners: the halo x halo corner)."""
    ni, nj, _ = decomp.local_domain
    hi, hj = halo
    out = []
    for d, (di, dj) in enumerate(DIRS8):
        nb = decomp.neighbour(di, dj)
        if nb is None:
            continue
        i0, i1 = {-1: (0, hi), 0: (0, ni), 1: (ni - hi, ni)}[di]
        j0, j1 = {-1: (0, hj), 0: (0, nj), 1: (nj - hj, nj)}[dj]
        out.append((d, nb, (max(i0, 0), min(i1, ni), max(j0, 0), min(j1, nj))))
    return out


def mirror_descriptor(me: Decomposition, nb: Decomposition, box: tuple, nb_base: int, nb_strides: tuple,
                      nb_origin: tuple, itemsize: int) -> tuple:
    """One ``Module.set_mirror`` box: our local cells ``box`` = (i0, i1, j0, j1)
    go to the neighbour's storage (element [0,0,0] at ``nb_base``, element
    strides ``nb_strides``, compute-domain origin ``nb_origin``): local (i, j, k)
    -> neighbour storage element origin + (I0 - nI0 + i, J0 - nJ0 + j, k)."""
    si, sj, sk = nb_strides
    oi, oj, ok = nb_origin
    off = (oi + me.i0 - nb.i0) * si + (oj + me.j0 - nb.j0) * sj + ok * sk
    return (*box, nb_base + off * itemsize, si, sj, sk)


class PeerFusedStep:
    """One decomposed time step in ONE kernel launch: the producing kernel
    itself stores the boundary values of its output into the neighbours'
    halos (peer memory: NVLink / NVSwitch between GPUs, CUDA IPC within one),
    so there is no separate exchange, pack or copy -- the transfer overlaps
    the computation tile by tile (the dycore step, one halo
    exchange per step, fused into the producer).

    ``phases``: field bindings cycled step by step (the dycore's u_in / u_out
    swap: ``[{u_in: A, u_out: B, ...}, {u_in: B, u_out: A, ...}]``); the
    stencil is compiled with ``gen_options={"mirror": out_field}`` so its
    column kernel stores ``out_field`` also through the mirror boxes
    (``Module.set_mirror``: up to 8 neighbours, corners included, each cell
    sent by its owner).  Per step, on one stream: wait until every neighbour
    finished its previous step (``gts_b200_flags_wait_next``: its stores into
    our input's halo are complete, and it no longer reads the halo of the
    buffer we are about to write into), launch, then bump every neighbour's
    counter (``gts_b200_flags_add``).  The result is bitwise the undecomposed
    run's (the same instructions per point; halos arrive before they are
    read)."""

    def __init__(self, stencil, decomposition: Decomposition, phases: list, scalars: dict,
                 out_field: str, halo: tuple, group=None, stream: Optional[int] = None, _local=False):
        import ctypes

        from . import native

        self._prepare(stencil, decomposition, phases, scalars, out_field, halo, stream)
        if _local:  # PeerFusedStep.local_group connects the virtual ranks itself
            return
        import torch.distributed as dist

        single = tuple(decomposition.grid) == (1, 1)  # no neighbours, no process group needed
        allv = []
        if not single:
            def handle(ptr):
                h, off = ctypes.create_string_buffer(64), ctypes.c_size_t()
                native.call("gts_b200_ipc_get_handle", ptr, h, ctypes.byref(off))
                return h.raw, off.value

            me = {"outs": [(handle(f.base_address()), tuple(f.strides), tuple(f.origin)) for f in self._outs],
                  "flags": handle(self._flags.dptr), "box": (decomposition.i0, decomposition.j0)}
            allv = [None] * dist.get_world_size(group)
            dist.all_gather_object(allv, me, group=group)

        def ipc_open(h):
            p = ctypes.c_void_p()
            native.call("gts_b200_ipc_open", h, ctypes.byref(p))
            self._opened.append(p.value)
            return p.value

        self._connect(allv, ipc_open)
        if not single:
            dist.barrier(group)  # every rank mapped its peers
            # the initial halos are valid and no buffer is being read: one
            # arrival per neighbour lets everyone's first step start
            native.call("gts_b200_flags_add", self._remote_arr, self._n, self.stream)
            native.synchronize(self.stream)
            dist.barrier(group)

    def _prepare(self, stencil, decomposition, phases, scalars, out_field, halo, stream) -> None:
        """This rank's own state: flags, expected counts, its output storages."""
        from . import native, storage

        module = stencil.build_info["module"]
        if getattr(module, "_mirror_fn", None) is None:
            raise ValueError(f"compile the stencil with gen_options={{'mirror': '{out_field}'}}")
        self.native, self.module, self.decomp = native, module, decomposition
        self.stream = native.default_stream() if stream is None else stream
        self.phases = phases
        self.out_field = out_field
        self._scalars, self._halo = scalars, halo
        self._flags = storage._DeviceBuffer(64, pinned_host=False)  # ARRIVED[8], one per direction
        self._expect = storage._DeviceBuffer(64, pinned_host=False)
        native.call("gts_b200_memset", self._flags.dptr, 0, 64, self.stream)
        native.call("gts_b200_memset", self._expect.dptr, 0, 64, self.stream)
        native.synchronize(self.stream)
        outs = []  # distinct output storages across phases, shared with the neighbours
        for ph in phases:
            f = ph[out_field]
            if not isinstance(f, storage.DeviceFieldStorage):
                raise TypeError("PeerFusedStep needs DeviceFieldStorages")
            if all(f is not o for o in outs):
                outs.append(f)
        self._outs = outs
        self._opened = []

    def _connect(self, allv: list, open_fn) -> None:
        """Map every neighbour's flags and outputs (``allv[rank]``: its
        ``outs`` / ``flags`` handles and box origin; ``open_fn`` turns a
        handle into a device pointer: CUDA IPC between processes, the
        pointer itself within one) and build the per-phase mirror boxes and
        launchers."""
        import ctypes

        decomposition, module = self.decomp, self.module
        dom = decomposition.local_domain
        self.neighbours = mirror_boxes(decomposition, self._halo)
        remote_outs, self._remote_flags, self._my_flags = {}, [], []
        for d, nb, box in self.neighbours:
            info = allv[nb]
            gp = open_fn(info["flags"][0])
            opp = DIRS8.index(tuple(-x for x in DIRS8[d]))
            self._remote_flags.append(gp + info["flags"][1] + 8 * opp)
            self._my_flags.append(self._flags.dptr + 8 * d)
            for oi, ((h, off), strides, origin) in enumerate(info["outs"]):
                remote_outs[(d, oi)] = (open_fn(h) + off, strides, origin, info["box"])
        n = len(self.neighbours)
        self._n = n
        self._remote_arr = (ctypes.c_void_p * max(1, n))(*self._remote_flags)
        self._my_arr = (ctypes.c_void_p * max(1, n))(*self._my_flags)
        # per phase: the mirror boxes into the neighbours' copy of that phase's output
        self._boxes, self._launch = [], []
        item = self._outs[0].itemsize
        for ph in self.phases:
            oi = next(x for x, f in enumerate(self._outs) if f is ph[self.out_field])
            boxes = []
            for d, nb, box in self.neighbours:
                base, strides, origin, _ = remote_outs[(d, oi)]
                nbd = Decomposition(decomposition.global_domain, decomposition.grid, nb)
                boxes.append(mirror_descriptor(decomposition, nbd, box, base, strides, origin, item))
            self._boxes.append(boxes)
            self._launch.append(module.launcher(dom, ph, self._scalars, self.stream))
        self._step = 0

    @classmethod
    def local_group(cls, stencil, decompositions: list, phases: list, scalars: dict, out_field: str,
                    halo: tuple, streams: list) -> list:
        """All ranks of a decomposition as virtual ranks of ONE process on one
        GPU, each on its own stream (``phases[r]``, ``streams[r]``): the same
        kernels, mirror stores and step flags as across GPUs, with the
        neighbours' outputs and flags addressed directly instead of through
        CUDA IPC.  The ranks' kernels run concurrently (no context
        time-slicing), so the step time shows the protocol's cost on
        hardware; it is not a scaling number (the ranks share one GPU)."""
        steps = [cls(stencil, d, ph, scalars, out_field, halo, stream=st, _local=True)
                 for d, ph, st in zip(decompositions, phases, streams)]
        allv = [{"outs": [((f.base_address(), 0), tuple(f.strides), tuple(f.origin)) for f in s_._outs],
                 "flags": (s_._flags.dptr, 0), "box": (s_.decomp.i0, s_.decomp.j0)} for s_ in steps]
        for s_ in steps:
            s_._connect(allv, lambda h: h)
        for s_ in steps:
            s_.native.call("gts_b200_flags_add", s_._remote_arr, s_._n, s_.stream)
        for s_ in steps:
            s_.native.synchronize(s_.stream)
        return steps

    def __call__(self) -> None:
        p = self._step % len(self.phases)
        self.native.call("gts_b200_flags_wait_next", self._my_arr, self._expect.dptr, self._n, self.stream)
        self.module.set_mirror(self._boxes[p])
        self._launch[p]()
        self.native.call("gts_b200_flags_add", self._remote_arr, self._n, self.stream)
        self._step += 1

    def graph(self, steps: int):
        """``steps`` steps (a multiple of the phase count, so every replay
        starts at the same phase) captured into one CUDA graph."""
        if steps % len(self.phases) or self._step % len(self.phases):
            raise ValueError(f"capture at phase 0, a multiple of {len(self.phases)} steps")
        upload_pending([st for ph in self.phases for st in ph.values()], self.stream)
        g = self.native.Graph(self.stream)
        start = self._step
        with g.capture():
            for _ in range(steps):
                self()
        self._step = start
        outs = [ph[self.out_field] for ph in self.phases]
        outer = self

        class _Replay:
            graph = g

            def launch(self_) -> None:
                if outer._step % len(outer.phases):
                    raise RuntimeError("replay must start at phase 0")
                g.launch()
                outer._step += steps
                for f in outs:  # written here and by the neighbours: host mirrors are stale
                    f.mark_device_written()

        return _Replay()

    def close(self) -> None:
        for p in self._opened:
            try:
                self.native.call("gts_b200_ipc_close", p)
            except Exception:  # pragma: no cover - teardown
                pass
        self._opened = []
