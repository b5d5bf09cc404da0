"""nvcc toolchain probe and the fingerprint-keyed module cache.

Mirrors the reference gen engine's build protocol (stencilforge
``backends/gen.py:64-103, 377-447, 458-466``) for sm_100a CUDA modules:

* ``toolchain_version()`` -- "nvcc <release> | sm_100a | <flags>", a
  fingerprint input exactly like gen's toolchain string (``runtime.py:305``);
* ``BuildCache`` -- ``<root>/<digest>/{source.cu, module.so, meta.json}``,
  immutable entries published by an atomic directory rename; a corrupt entry
  is evicted and rebuilt once; ``COMPILER_INVOCATIONS`` counts real nvcc runs.

The default cache root is in-tree (``paper_2311_08322_b200/_cache``) so that
modules prebuilt by ``__graft_entry__.build()`` travel with the repository
snapshot to the GPU box; ``GTS_B200_CACHE_DIR`` overrides it.
"""

from __future__ import annotations

import ctypes
import json
import os
import shutil
import subprocess
import time
import uuid
from pathlib import Path
from typing import Optional

from ._host import BackendError, Code

PKG = Path(__file__).resolve().parent
TEMPLATES = PKG / "csrc" / "templates"
DEFAULT_CACHE = PKG / "_cache"

COMPILER_INVOCATIONS = 0
_PROBE: dict = {}

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_command() -> str:
    env = os.environ.get("GTS_NVCC")
    if env:
        return env
    cand = Path("/usr/local/cuda/bin/nvcc")
    return str(cand) if cand.exists() else "nvcc"


def compile_flags() -> list:
    # --fmad=false keeps arithmetic bitwise-aligned with the reference engines
    # (gen compiles with -ffp-contract=off, gen.py:64-67); IEEE division and
    # square root and no flush-to-zero are nvcc's defaults, spelled out.
    return [
        "-O3", "-std=c++17", *ARCH_FLAGS, "-lineinfo", "--fmad=false",
        "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
        "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-warn-spills",
    ]


def cache_root() -> Path:
    env = os.environ.get("GTS_B200_CACHE_DIR")
    return Path(env) if env else DEFAULT_CACHE


def toolchain_version() -> str:
    nvcc = nvcc_command()
    if nvcc in _PROBE:
        return _PROBE[nvcc]
    try:
        out = subprocess.run([nvcc, "--version"], capture_output=True, text=True, timeout=60)
    except (OSError, subprocess.TimeoutExpired) as exc:
        raise BackendError(Code.TOOLCHAIN_MISSING, f"cannot run '{nvcc} --version': {exc}")
    if out.returncode != 0:
        raise BackendError(Code.TOOLCHAIN_MISSING, f"'{nvcc} --version' failed: {out.stderr.strip()}")
    release = [ln for ln in out.stdout.splitlines() if "release" in ln]
    version = release[0].strip() if release else out.stdout.strip().splitlines()[-1]
    _PROBE[nvcc] = (f"nvcc | {version} | sm_100a | {' '.join(compile_flags())} | "
                    f"codegen {codegen_digest()}")
    return _PROBE[nvcc]


def codegen_digest() -> str:
    """Content hash of the lowering, code generators and templates: part of
    the toolchain string, so a generator change can never serve a stale
    module from the cache."""
    import hashlib

    h = hashlib.sha256()
    files = sorted(PKG.glob("codegen*.py")) + [PKG / "lowering.py"] + sorted(TEMPLATES.glob("*.cuh"))
    for f in files:
        h.update(f.name.encode())
        h.update(f.read_bytes())
    return h.hexdigest()[:12]


def _invoke_nvcc(src: Path, so: Path) -> None:
    global COMPILER_INVOCATIONS
    nvcc = nvcc_command()
    cmd = [nvcc, *compile_flags(), f"-I{TEMPLATES}", str(src), "-o", str(so)]
    COMPILER_INVOCATIONS += 1
    env = dict(os.environ)
    env.pop("CC", None)  # a CC wrapper without libgomp must not leak into nvcc -ccbin
    try:
        proc = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    except OSError as exc:
        raise BackendError(Code.TOOLCHAIN_MISSING, f"cannot run '{nvcc}': {exc}")
    if proc.returncode != 0:
        raise BackendError(Code.COMPILE_FAILED, f"{' '.join(cmd)} failed:\n{proc.stderr.strip()}")


class BuildCache:
    """Fingerprint-keyed store of generated CUDA sources and modules."""

    def __init__(self, root: Optional[os.PathLike] = None):
        self.root = Path(root) if root is not None else cache_root()
        self.root.mkdir(parents=True, exist_ok=True)

    def entry_dir(self, fp) -> Path:
        return self.root / fp.digest

    def so_path(self, fp) -> Path:
        return self.entry_dir(fp) / "module.so"

    def source_path(self, fp) -> Path:
        return self.entry_dir(fp) / "source.cu"

    def lookup(self, fp) -> Optional[Path]:
        so = self.so_path(fp)
        return so if so.is_file() else None

    def evict(self, fp) -> None:
        shutil.rmtree(self.entry_dir(fp), ignore_errors=True)

    def install(self, fp, source: str, stencil_name: str, plan: Optional[list] = None) -> Path:
        tmp = self.root / f".build-{fp.short}-{os.getpid()}-{uuid.uuid4().hex[:8]}"
        tmp.mkdir(parents=True)
        try:
            src = tmp / "source.cu"
            src.write_text(source)
            _invoke_nvcc(src, tmp / "module.so")
            meta = {
                "fingerprint": fp.digest,
                "stencil": stencil_name,
                "toolchain": toolchain_version(),
                "plan": plan or [],
                "created": time.time(),
            }
            (tmp / "meta.json").write_text(json.dumps(meta, indent=2))
            try:
                os.rename(tmp, self.entry_dir(fp))
            except OSError:
                if self.lookup(fp) is None:
                    # a stale entry without its object (a crashed or pruned
                    # build): replace it, still by one atomic rename
                    self.evict(fp)
                    os.rename(tmp, self.entry_dir(fp))
        finally:
            shutil.rmtree(tmp, ignore_errors=True)
        return self.so_path(fp)


_OBJECT_MAGIC = b"\x7fELF"


def load_library(so: Path) -> ctypes.CDLL:
    """dlopen after a header check (a cached corrupt object must be detected
    before dlopen hands back a stale mapping, gen.py:458-466)."""
    with open(so, "rb") as f:
        if f.read(4) != _OBJECT_MAGIC:
            raise OSError(f"{so} is not a loadable object")
    return ctypes.CDLL(str(so))
