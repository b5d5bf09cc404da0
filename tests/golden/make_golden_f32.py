"""Generate tests/golden/corpus_f32.npz: binary32 variants of the reference
corpus programs, run by the reference's own ``debug`` engine.

The reference corpus (corpus.generate_corpus(seed=2024), test_acceptance.py:
34-35, 116-129) is all-f64.  Its f32 storage semantics (binary64 arithmetic,
every store narrowed; debug.py / vec.py, gen.py:276-277 for scalars aside)
are what the b200 backend's binary32-exact rewrites (codegen.emit_f32*) must
reproduce, so this script takes the first N programs of corpus.json, declares
every field ``Field[f32]``, feeds the seeded inputs of tests/_inputs.py, and
stores the debug engine's output compute views (small domains, stored in
full: NaN payloads differ between NumPy and the GPU, so the GPU test compares
NaN masks plus the bits of every other element).  ``vec`` is checked equal.

Run here (needs /root/reference):  python tests/golden/make_golden_f32.py
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("GTS_CACHE_DIR", tempfile.mkdtemp(prefix="gts-golden-"))

import stencilforge as sf  # noqa: E402

import _inputs  # noqa: E402

N = 120


def f32_source(src: str) -> str:
    return src.replace("Field[f64]", "Field[f32]")


def main():
    meta = json.loads((HERE / "corpus.json").read_text())[:N]
    out = {}
    names = []
    for e in meta:
        src = f32_source(e["source"])
        dom = tuple(e["domain"])
        res = {}
        for backend in ("debug", "vec"):
            st = sf.compile_stencil(src, e["name"], backend=backend)
            arrays = _inputs.random_field_arrays(st.implementation, dom, np.random.default_rng(e["seed"]))
            lay = sf.default_layout(backend)
            fields = {n: sf.from_array(arr, origin, lay) for n, (arr, origin) in arrays.items()}
            st(domain=dom, **fields, **e["scalars"])
            res[backend] = {o: np.asarray(fields[o].compute_view(dom)).copy() for o in e["outputs"]}
        for o in e["outputs"]:
            a, b = res["debug"][o], res["vec"][o]
            assert a.dtype == np.float32
            assert np.array_equal(a, b, equal_nan=True), (e["name"], o)
            out[f"{e['name']}_{o}"] = a
        names.append(e["name"])
    np.savez_compressed(HERE / "corpus_f32.npz", **out)
    print("programs", len(names), "arrays", len(out), (HERE / "corpus_f32.npz").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
