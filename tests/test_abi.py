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
