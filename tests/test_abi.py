"""The C-ABI boundary (include/gts_b200.h) without a GPU: libraries load and
export every declared symbol; generated modules follow the gen mangling and
argument convention; the module cache follows the gen BuildCache protocol."""

import ctypes
import re
from pathlib import Path

import pytest

import paper_2311_08322_b200 as b200
from paper_2311_08322_b200 import native, toolchain, workloads

REPO = Path(__file__).resolve().parent.parent
HEADER = REPO / "include" / "gts_b200.h"


def declared(prefix):
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(" + prefix + r"\w+)\s*\(", text)))


def test_runtime_library_exports_header_symbols():
    lib = native.lib()
    names = [n for n in declared("gts_b200_") if not n.startswith("gts_b200_module_")]
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert lib.gts_b200_abi_version() == 1
    assert set(native.SIGNATURES) == set(names)


def test_error_strings():
    assert native.error_string(1001).startswith("vertical domain")
    assert native.error_string(0) == "success"


@pytest.mark.parametrize("kernel,dtype", [("hdiff", "f64"), ("hdiff", "f32"), ("vadv", "f64"), ("vadv", "f32")])
def test_prebuilt_modules_export_entry(kernel, dtype):
    before = toolchain.COMPILER_INVOCATIONS
    st = b200.compile_stencil(workloads.source(kernel, dtype), kernel)
    assert st.backend == "b200"
    assert st.build_info["arch"] == "sm_100a"
    so = st.build_info["so_path"]
    lib = ctypes.CDLL(so)
    sym = st.build_info["symbol"]
    assert sym == f"gts_run_{kernel}_{st.fingerprint.short}"
    assert hasattr(lib, sym)
    for n in declared("gts_b200_module_"):
        assert hasattr(lib, n), n
    if kernel == "hdiff":  # a single fused PARALLEL kernel: frame launch + its tile shape
        short = st.fingerprint.short
        assert hasattr(lib, f"gts_frame_{kernel}_{short}")
        ft = getattr(lib, f"gts_frametile_{kernel}_{short}")
        ft.restype = ctypes.c_int
        assert (ft() >> 16, ft() & 0xFFFF) == st.build_info["module"].frame_tile == (4, 32)
    # prebuilt by __graft_entry__.build(): served from the in-tree cache
    assert toolchain.COMPILER_INVOCATIONS == before
    assert st.build_info["cache_hit"] is True


def test_fingerprint_uses_b200_backend_id_and_nvcc_toolchain():
    st = b200.compile_stencil(workloads.source("hdiff"), "hdiff")
    import stencilforge as sf

    gen = sf.compile_stencil(workloads.source("hdiff"), "hdiff", backend="debug")
    assert st.fingerprint != gen.fingerprint
    assert "nvcc" in toolchain.toolchain_version() and "sm_100a" in toolchain.toolchain_version()


def test_non_b200_backends_forwarded_to_reference():
    st = b200.compile_stencil(workloads.source("hdiff"), "hdiff", backend="vec")
    assert st.backend == "vec"


def test_sass_has_no_fma_for_parity_build():
    """--fmad=false: the parity build must not contract into DFMA."""
    st = b200.compile_stencil(workloads.source("hdiff"), "hdiff")
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", st.build_info["so_path"]],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "DFMA" not in out.stdout
    assert "DADD" in out.stdout and "DMUL" in out.stdout


class _FakeCAI:
    def __init__(self, shape, strides, typestr="<f8"):
        self.__cuda_array_interface__ = {"shape": shape, "strides": strides, "typestr": typestr,
                                         "data": (0x1000, False), "version": 3}


@pytest.mark.parametrize("shape,strides,typestr", [
    ((4, 5), None, "<f8"),                        # not 3-D
    ((4, 5, 6), None, "<i4"),                     # element type
    ((4, 5, 6), None, "<f8"),                     # C order: k contiguous, not the b200 axis order
    ((4, 5, 6), (40, 8, 12), "<f8"),              # strides not element multiples
    ((4, 5, 6), (48, 8, 160), "<f8"),             # s_k < s_i * ni
])
def test_from_cuda_array_rejects_bad_arrays(shape, strides, typestr):
    """Zero-copy wrapping validates shape / dtype / axis order before touching
    the device (storage.ExternalDeviceFieldStorage)."""
    from paper_2311_08322_b200.storage import StorageError

    with pytest.raises(StorageError):
        b200.from_cuda_array(_FakeCAI(shape, strides, typestr))


@pytest.mark.parametrize("ni", [128, 129, 150, 200, 256, 511, 512, 1000, 2048])
def test_pipeline_chunks_cover_rows(ni):
    """backend._Pipeline.chunk_bounds: contiguous cover of [0, ni), CHUNK_ROWS
    pieces then a taper, no piece below 16 rows."""
    from paper_2311_08322_b200.backend import _Pipeline

    b = _Pipeline.chunk_bounds(ni)
    assert b[0][0] == 0 and b[-1][1] == ni
    assert all(x1 == y0 for (_, x1), (y0, _) in zip(b, b[1:]))
    sizes = [y - x for x, y in b]
    assert all(s >= 16 for s in sizes) and max(sizes) <= _Pipeline.CHUNK_ROWS + 15
    body = sizes[:-1]  # the last piece absorbs a remainder below 16 rows
    assert body == sorted(body, reverse=True)


def test_execution_report_extends_reference_report():
    """B200ExecutionReport is the reference's ExecutionReport (runtime.py:21-38)
    with device time and bytes moved added to as_dict()."""
    import stencilforge as sf
    from paper_2311_08322_b200.api import B200ExecutionReport

    r = B200ExecutionReport(10, 2, 5, (4, 4, 4), True, 3000, 2000, 64, 32)
    assert isinstance(r, sf.ExecutionReport)
    d = r.as_dict()
    assert d["kernel_ns"] == 5 and d["device_ns"] == 3000 and d["h2d_bytes"] == 64 and d["d2h_bytes"] == 32


def test_binary32_rewrites_in_generated_source():
    """codegen.emit_f32*: the f32 hdiff tile kernel computes the flux-limiter
    sign test with float comparisons and flx / fly as single binary32
    subtractions; the f64 kernel keeps its binary64 multiply; f32x=False
    restores the plain form (SURVEY.md 8(a) numerics)."""
    import re

    def src(dtype, opts=None):
        st = b200.compile_stencil(workloads.source("hdiff", dtype), "hdiff", gen_options=opts)
        return Path(st.build_info["source_path"]).read_text()

    s32 = src("f32")
    assert re.search(r"\(\(\(wf_lap\[\d\]\[\d\] > wf_lap\[\d\]\[\d\]\) && \(wf_inp", s32)
    assert re.search(r"const float vf_ = \(wf_lap\[\d\]\[\d\] - wf_lap\[\d\]\[\d\]\);", s32)
    s64 = src("f64")
    assert "wf_" not in s64 and "> 0x0.0p+0" in s64
    plain = src("f32", {"f32x": False})
    assert "wf_" not in plain


def test_f32_exact_literals():
    from paper_2311_08322_b200.codegen import _f32_exact_literal

    assert _f32_exact_literal(0.0) and _f32_exact_literal(4.0) and _f32_exact_literal(-0.5)
    assert not _f32_exact_literal(0.1) and not _f32_exact_literal(1e300)
    assert not _f32_exact_literal(float("nan")) and not _f32_exact_literal(float("inf"))


def test_bench_reference_arm_contract():
    """bench.py --impl reference (the reference's own CPU kernel, oracle/_ref,
    on the host cores): one JSON line with the arm's keys, e2e with zero
    host<->device bytes, and the arena-reuse secondary row."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    repo = Path(__file__).resolve().parent.parent
    if not (repo / "oracle" / "_ref" / "manifest.json").exists():
        pytest.skip("oracle/_ref not built (run __graft_entry__.build())")
    r = subprocess.run([sys.executable, str(repo / "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=str(repo))
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "grid-points/s" and line["higher_is_better"] is True
    assert line["steps"] == 2 and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert cb["rows"]["gen_arena_reuse"]["value"] > 0


def test_l2_prefetch_before_griddep_wait_in_generated_source():
    """Round-2 L2 prefetch (K2 "L2 prefetch"): the vadv column
    kernel and the hdiff tile kernel prefetch their first tile into L2 before
    griddepcontrol.wait, the column kernel also after the second tile's ring
    fill; the fused dycore kernel (prologue) and explicit opt-outs do not."""

    def kernel_body(kernel, dtype, name, opts=None):
        st = b200.compile_stencil(workloads.source(kernel, dtype), kernel, gen_options=opts)
        src = Path(st.build_info["source_path"]).read_text()
        m = re.search(r"__global__ void __launch_bounds__\([^)]*\) " + name + r"\(", src)
        assert m, name
        end = src.find("\n__global__", m.end())
        return src[m.end():end if end > 0 else len(src)]

    for kernel, dtype, name in (("vadv", "f64", "gts_k0_column_tmem_w1s4c2"), ("vadv", "f64", "gts_k0_column_tmem_w2"),
                                ("hdiff", "f64", "gts_k0_pfused"),
                                ("hdiff", "f32", "gts_k0_pfused")):
        body = kernel_body(kernel, dtype, name)
        pf, wait = body.find("gts_tma_prefetch_l2_3d"), body.find("gts_griddep_wait()")
        assert 0 <= pf < wait, (kernel, dtype)
    body = kernel_body("vadv", "f64", "gts_k0_column_tmem_w2")
    assert "ntiles <= 2 * (int)gridDim.x" in body
    off = kernel_body("vadv", "f64", "gts_k0_column_tmem_w2", {"col_l2pf0": 0, "col_l2pf": 0})
    assert "gts_tma_prefetch_l2_3d" not in off
    assert "gts_tma_prefetch_l2_3d" not in kernel_body("dycore", "f64", "gts_k1_column_tmem_w2s4")


def test_pin_in_place_bookkeeping_leaves_with_the_buffer(monkeypatch):
    """backend._pin_host_buffer: a buffer that needs no pinning (already
    page-locked) or could not be pinned must not leave a stale entry behind
    once it is freed -- a later pageable buffer that reuses its id() would
    otherwise never be page-locked (its copies fall back to the driver's
    staged path: 3.6 -> 5.7 ms per vadv call measured)."""
    import gc

    import numpy as np

    from paper_2311_08322_b200 import backend

    calls = []

    class _Lib:
        def gts_b200_host_register(self, ptr, nbytes, reg):
            calls.append(ptr)
            return 0  # "already page-locked": success, nothing registered

        def gts_b200_host_unregister(self, ptr):  # pragma: no cover - must not be called
            raise AssertionError("unregistered a buffer it did not register")

    monkeypatch.setattr(backend.native, "lib", lambda: _Lib())
    a = np.zeros(1024)
    key = id(a)
    backend._pin_host_buffer(a)
    backend._pin_host_buffer(a)  # cached while alive
    assert key in backend._pinned_in_place and backend._pinned_in_place[key] is False and len(calls) == 1
    del a
    gc.collect()
    assert key not in backend._pinned_in_place


def test_bench_conversion_roofline_from_sass(monkeypatch):
    """bench.conversion_roofline: the f32 hdiff tile kernel's binary32 <->
    binary64 conversions per point come from the module's SASS (the fully
    unrolled thread-tile body), 7.75 with the default geometry,
    and the fraction is taken against 16 conversions /clk/SM."""
    import shutil
    import sys

    if not (shutil.which("cuobjdump") or Path("/usr/local/cuda/bin/cuobjdump").exists()):
        pytest.skip("cuobjdump unavailable")
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench

    monkeypatch.setattr(native, "device_info", lambda dev=None: {"sm_count": 148})

    class _S:
        def summary(self):
            return {"sm_mhz": 1965.0}

    st = b200.compile_stencil(workloads.source("hdiff", "f32"), "hdiff")
    r = bench.conversion_roofline(st, (256, 256, 80), 13.7e-6, _S())
    assert r["conv_per_point"] == 7.75
    assert abs(r["peak"] - 16 * 148 * 1965e6 / 1e12) < 1e-9
    assert 0.6 < r["frac"] < 0.7
