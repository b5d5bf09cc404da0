"""Generate the committed golden fixtures by running the REFERENCE itself.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

Outputs (all small, committed):
  kernels.npz   hdiff / vadv inputs + outputs of the reference's ``vec``
                backend, its ``debug`` backend (small cases) and its
                independent oracles (oracles.py:15-78), f64 and f32.
  corpus.json   the first N programs of the reference's differential corpus
                (corpus.generate_corpus(seed=2024), test_acceptance.py:34-35,
                116-129): source, domain, seed, SHA-256 of every input
                storage (to pin tests/_inputs.py's restatement of
                corpus.random_field_args) and of every output compute view
                produced by the reference ``debug`` backend (bitwise).
  corpus_out.npz full output compute views for the programs with
                ``"stored": true`` so max_rel can be reported, not just a hash.
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
from stencilforge import corpus  # noqa: E402
from stencilforge.kernels import kernel_source  # noqa: E402
from stencilforge.oracles import hdiff_reference, make_diagonally_dominant, vadv_reference  # noqa: E402

import _inputs  # noqa: E402

CORPUS_N = 200
CORPUS_STORED = 40
CORPUS_DOMAINS = [(4, 4, 6), (8, 7, 5), (16, 16, 16), (6, 12, 9), (16, 8, 4), (5, 5, 16)]
VADV_RANGES = {"a": (0.1, 0.45), "c": (0.1, 0.45), "b": (1.0, 2.0), "d": (-1.0, 1.0)}

HDIFF32 = kernel_source("hdiff").replace("Field[f64]", "Field[f32]")
VADV32 = kernel_source("vadv").replace("Field[f64]", "Field[f32]")


def run_ref(backend, source, name, arrays, origins, scalars, domain=None):
    st = sf.compile_stencil(source, name, backend=backend)
    layout = sf.default_layout(backend)
    fields = {n: sf.from_array(arrays[n], origins[n], layout) for n in arrays}
    st(domain=domain, **fields, **scalars)
    return {n: np.asarray(fields[n].data()).copy() for n in arrays}


def kernels_npz():
    out = {}
    # hdiff f64: the reference's own oracle-test domains and seeds
    # (test_kernels.py:25-32, test_acceptance.py:160-169) + bench seed 0.
    for dom in [(8, 8, 8), (16, 16, 16), (32, 32, 8), (13, 9, 5)]:
        rng = np.random.default_rng(sum(dom))
        inp = rng.uniform(-1, 1, (dom[0] + 4, dom[1] + 4, dom[2]))
        key = "hdiff_f64_%dx%dx%d" % dom
        arrays = {"inp": inp, "out": np.zeros(dom)}
        origins = {"inp": (2, 2, 0), "out": (0, 0, 0)}
        vec = run_ref("vec", kernel_source("hdiff"), "hdiff", arrays, origins, {"coeff": 0.05})
        dbg = run_ref("debug", kernel_source("hdiff"), "hdiff", arrays, origins, {"coeff": 0.05})
        assert np.array_equal(vec["out"], dbg["out"])
        out[key + "_inp"] = inp
        out[key + "_out"] = vec["out"]
        out[key + "_nested"] = hdiff_reference(inp, 0.05)
    # hdiff f32 (f32 storage and temporaries, f64 arithmetic)
    for dom in [(16, 16, 16), (9, 14, 3)]:
        rng = np.random.default_rng(1000 + sum(dom))
        inp = rng.uniform(-1, 1, (dom[0] + 4, dom[1] + 4, dom[2])).astype(np.float32)
        key = "hdiff_f32_%dx%dx%d" % dom
        arrays = {"inp": inp, "out": np.zeros(dom, np.float32)}
        origins = {"inp": (2, 2, 0), "out": (0, 0, 0)}
        vec = run_ref("vec", HDIFF32, "hdiff", arrays, origins, {"coeff": 0.05})
        dbg = run_ref("debug", HDIFF32, "hdiff", arrays, origins, {"coeff": 0.05})
        assert np.array_equal(vec["out"], dbg["out"])
        out[key + "_inp"] = inp
        out[key + "_out"] = vec["out"]
    # vadv f64: K in {1, 3, 8, 80} with the reference's seeds (test_acceptance.py:133-158)
    for nk in (1, 3, 8, 80):
        dom = (10, 10, nk)
        rng = np.random.default_rng(300 + nk)
        a, b, c, d = make_diagonally_dominant(rng, dom)
        key = "vadv_f64_%dx%dx%d" % dom
        arrays = {"a": a, "b": b, "c": c, "d": d, "x": np.zeros(dom)}
        origins = {n: (0, 0, 0) for n in arrays}
        vec = run_ref("vec", kernel_source("vadv"), "vadv", arrays, origins, {})
        for n, v in zip("abcd", (a, b, c, d)):
            out[f"{key}_{n}"] = v
        out[key + "_x"] = vec["x"]
        out[key + "_dense"] = vadv_reference(a, b, c, d)
        if nk <= 8:
            dbg = run_ref("debug", kernel_source("vadv"), "vadv", arrays, origins, {})
            assert np.array_equal(vec["x"], dbg["x"])
    for nk in (1, 6, 33):
        dom = (7, 11, nk)
        rng = np.random.default_rng(500 + nk)
        a, b, c, d = (v.astype(np.float32) for v in make_diagonally_dominant(rng, dom))
        key = "vadv_f32_%dx%dx%d" % dom
        arrays = {"a": a, "b": b, "c": c, "d": d, "x": np.zeros(dom, np.float32)}
        origins = {n: (0, 0, 0) for n in arrays}
        vec = run_ref("vec", VADV32, "vadv", arrays, origins, {})
        for n, v in zip("abcd", (a, b, c, d)):
            out[f"{key}_{n}"] = v
        out[key + "_x"] = vec["x"]
    np.savez_compressed(HERE / "kernels.npz", **out)


def corpus_fixtures():
    progs = corpus.generate_corpus(seed=2024, count=CORPUS_N)
    meta = []
    stored = {}
    for idx, p in enumerate(progs):
        domain = CORPUS_DOMAINS[idx % len(CORPUS_DOMAINS)]
        seed = 50_000 + idx  # test_acceptance.py:118
        st = sf.compile_stencil(p.source, p.name, backend="debug")
        impl = st.implementation
        # reference inputs
        rng = np.random.default_rng(seed)
        fields = corpus.random_field_args(impl, "debug", domain, rng)
        scalars = corpus.random_scalar_args(impl, np.random.default_rng(seed + 1))
        # pin the restatement
        mine = _inputs.random_field_arrays(impl, domain, np.random.default_rng(seed))
        in_sha = {}
        for f in impl.api_fields:
            ref_arr = np.asarray(fields[f.name].data())
            arr, origin = mine[f.name]
            assert arr.shape == ref_arr.shape and origin == fields[f.name].origin
            assert np.array_equal(arr, ref_arr, equal_nan=True), (p.name, f.name)
            in_sha[f.name] = _inputs.sha(arr)
        assert _inputs.random_scalars(impl, np.random.default_rng(seed + 1)) == scalars
        st(domain=domain, **fields, **scalars)
        outs = {o: np.asarray(fields[o].compute_view(domain)).copy() for o in p.outputs}
        # vec must agree bitwise (criterion 1 is 1e-13; the ops used are exact)
        stv = sf.compile_stencil(p.source, p.name, backend="vec")
        fv = corpus.random_field_args(stv.implementation, "vec", domain, np.random.default_rng(seed))
        stv(domain=domain, **fv, **scalars)
        for o in p.outputs:
            assert np.array_equal(np.asarray(fv[o].compute_view(domain)), outs[o], equal_nan=True)
        entry = {
            "idx": idx, "name": p.name, "source": p.source, "domain": list(domain),
            "seed": seed, "outputs": list(p.outputs), "scalars": scalars,
            "input_sha": in_sha,
            "output_sha": {o: _inputs.sha(v) for o, v in outs.items()},
            "stored": idx < CORPUS_STORED,
        }
        if idx < CORPUS_STORED:
            for o, v in outs.items():
                stored[f"{p.name}_{o}"] = v
        meta.append(entry)
    (HERE / "corpus.json").write_text(json.dumps(meta, indent=1))
    np.savez_compressed(HERE / "corpus_out.npz", **stored)


if __name__ == "__main__":
    kernels_npz()
    corpus_fixtures()
    for f in ("kernels.npz", "corpus.json", "corpus_out.npz"):
        print(f, (HERE / f).stat().st_size)
