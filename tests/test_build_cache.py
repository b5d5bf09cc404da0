"""The fingerprint-keyed CUDA module cache: the b200
analogues of the reference's criterion 6 (test_acceptance.py:276-301), its
corrupt-object rebuild (test_backends.py:249-263) and its missing-compiler
check (test_backends.py:311-318).  CPU only (nvcc cross-compiles), each test
with its own temporary cache directory."""

import os

import pytest

import paper_2311_08322_b200 as b200
from paper_2311_08322_b200 import toolchain, workloads
from paper_2311_08322_b200._host import BackendError, Code

SCALED = (
    "stencil scaled(a: Field[f64], b: Field[f64]):\n"
    "    with computation(PARALLEL):\n"
    "        with interval(0, None):\n"
    "            b = a * K0\n"
)
COPY = (
    "stencil copy(a: Field[f64], b: Field[f64]):\n"
    "    with computation(PARALLEL):\n"
    "        with interval(0, None):\n"
    "            b = a\n"
)


def test_criterion_6_cache_behaviour(tmp_path):
    """A miss costs exactly one nvcc run; a reformatted source hits the same
    entry (0 compiles, same object path); a changed external rebuilds."""
    cache = str(tmp_path / "cache")
    src = workloads.source("hdiff")
    before = toolchain.COMPILER_INVOCATIONS
    st1 = b200.compile_stencil(src, "hdiff", cache_dir=cache)
    assert toolchain.COMPILER_INVOCATIONS == before + 1
    assert st1.build_info["cache_hit"] is False

    variant = "# reformatted\n" + src.replace(
        "out = inp - coeff", "out  =  inp  -  coeff"
    ).replace("with computation(PARALLEL):", "with computation(PARALLEL):  # body")
    assert variant != src
    st2 = b200.compile_stencil(variant, "hdiff", cache_dir=cache)
    assert toolchain.COMPILER_INVOCATIONS == before + 1, "reformatting recompiled"
    assert st2.build_info["cache_hit"] is True
    assert st1.build_info["so_path"] == st2.build_info["so_path"]

    b200.compile_stencil(SCALED, cache_dir=cache, externals={"K0": 1.0})
    mid = toolchain.COMPILER_INVOCATIONS
    b200.compile_stencil(SCALED, cache_dir=cache, externals={"K0": 1.0})
    assert toolchain.COMPILER_INVOCATIONS == mid, "identical external rebuilt"
    b200.compile_stencil(SCALED, cache_dir=cache, externals={"K0": 2.0})
    assert toolchain.COMPILER_INVOCATIONS == mid + 1, "changed external did not rebuild"


def test_corrupt_shared_object_is_rebuilt(tmp_path):
    """A cached module.so replaced by garbage is detected (ELF magic check
    before dlopen), evicted and rebuilt once."""
    cache = tmp_path / "cache"
    st1 = b200.compile_stencil(COPY, cache_dir=str(cache))
    so = st1.build_info["so_path"]
    garbage = tmp_path / "garbage.so"
    garbage.write_bytes(b"garbage not an elf")
    os.replace(garbage, so)  # replace, not overwrite: the first mapping stays valid
    before = toolchain.COMPILER_INVOCATIONS
    st2 = b200.compile_stencil(COPY, cache_dir=str(cache))
    assert toolchain.COMPILER_INVOCATIONS == before + 1
    assert st2.build_info["cache_hit"] is False
    with open(st2.build_info["so_path"], "rb") as f:
        assert f.read(4) == b"\x7fELF"
    # the entry is whole again: the next compile is a hit
    st3 = b200.compile_stencil(COPY, cache_dir=str(cache))
    assert st3.build_info["cache_hit"] is True
    assert toolchain.COMPILER_INVOCATIONS == before + 1


def test_half_written_entry_is_invisible(tmp_path):
    """Entries are published by an atomic directory rename: a leftover
    temporary build directory (a crashed build) is never served, and an entry
    directory without its object is a miss."""
    cache = tmp_path / "cache"
    st1 = b200.compile_stencil(COPY, cache_dir=str(cache))
    entry = os.path.dirname(st1.build_info["so_path"])
    os.remove(st1.build_info["so_path"])  # the entry lost its object
    (cache / ".build-deadbeef-1-00000000").mkdir()
    before = toolchain.COMPILER_INVOCATIONS
    st2 = b200.compile_stencil(COPY, cache_dir=str(cache))
    assert st2.build_info["cache_hit"] is False
    assert toolchain.COMPILER_INVOCATIONS == before + 1
    assert os.path.dirname(st2.build_info["so_path"]) == entry


def test_missing_compiler_reported(tmp_path, monkeypatch):
    """GTS_NVCC naming a missing compiler: BackendError TOOLCHAIN_MISSING
    (the reference's GTS_CC analogue) -- no CPU fallback, nothing cached."""
    monkeypatch.setenv("GTS_NVCC", "/nonexistent/bin/nvcc")
    toolchain._PROBE.clear()
    try:
        with pytest.raises(BackendError) as exc:
            b200.compile_stencil(COPY, cache_dir=str(tmp_path / "cache"))
        assert exc.value.code == Code.TOOLCHAIN_MISSING
        assert not any((tmp_path / "cache").glob("*/module.so"))
    finally:
        monkeypatch.delenv("GTS_NVCC")
        toolchain._PROBE.clear()


def test_compile_failure_reports_nvcc_stderr(tmp_path):
    """An nvcc error surfaces as COMPILE_FAILED with the compiler's message,
    and leaves no entry behind."""
    from paper_2311_08322_b200._host import analysis, ir
    from paper_2311_08322_b200.api import _select_definition

    cache = toolchain.BuildCache(tmp_path / "cache")
    bound = _select_definition(COPY, None, {}, None)
    impl = analysis.lower(bound)
    fp = ir.fingerprint(bound, "b200", {}, toolchain.toolchain_version(), {"broken": 1})
    with pytest.raises(BackendError) as exc:
        cache.install(fp, "this is not CUDA;\n", "copy")
    assert exc.value.code == Code.COMPILE_FAILED
    assert "error" in str(exc.value).lower()
    assert cache.lookup(fp) is None
    assert impl.name == "copy"
