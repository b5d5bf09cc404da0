"""Pin the oracle: both CPU restatements vs the reference's golden vectors
(tests/golden/make_golden.py ran the reference's own engines)."""

import json
from pathlib import Path

import numpy as np
import pytest

import _inputs
import oracle

GOLDEN = Path(__file__).parent / "golden"


def _cases(golden, prefix):
    return sorted({k.rsplit("_", 1)[0] for k in golden if k.startswith(prefix)})


def test_c_oracle_hdiff_bitwise(golden):
    for key in _cases(golden, "hdiff_"):
        got = oracle.hdiff_c(golden[key + "_inp"], 0.05)
        assert got.dtype == golden[key + "_out"].dtype
        assert np.array_equal(got, golden[key + "_out"]), key


def test_numpy_oracle_hdiff_bitwise(golden):
    for key in _cases(golden, "hdiff_"):
        got = oracle.hdiff_np(golden[key + "_inp"], 0.05)
        assert np.array_equal(got, golden[key + "_out"]), key


def test_hdiff_golden_vs_reference_nested_loop(golden):
    for key in _cases(golden, "hdiff_f64"):
        assert oracle.max_rel(golden[key + "_out"], golden[key + "_nested"]) <= 1e-14


def test_c_oracle_vadv_bitwise(golden):
    for key in _cases(golden, "vadv_"):
        a, b, c, d = (golden[f"{key}_{n}"] for n in "abcd")
        got = oracle.vadv_c(a, b, c, d)
        assert np.array_equal(got, golden[key + "_x"]), key
        got_np = oracle.vadv_np(a, b, c, d)
        assert np.array_equal(got_np, golden[key + "_x"]), key


def test_vadv_golden_vs_dense_solve(golden):
    for key in _cases(golden, "vadv_f64"):
        x, dense = golden[key + "_x"], golden[key + "_dense"]
        diff = np.max(np.abs(x - dense), axis=2)
        scale = np.maximum(np.max(np.abs(dense), axis=2), 1e-30)
        assert float(np.max(diff / scale)) <= 1e-12


@pytest.mark.parametrize("threads", [1, 2, 8])
def test_c_oracle_thread_count_invariant(threads):
    rng = np.random.default_rng(4)
    inp = rng.uniform(-1, 1, (36, 28, 9))
    assert np.array_equal(oracle.hdiff_c(inp, 0.05, threads), oracle.hdiff_np(inp, 0.05))


def test_input_restatement_matches_reference_hashes():
    """tests/_inputs.random_field_arrays reproduces corpus.random_field_args."""
    import paper_2311_08322_b200  # noqa: F401  (locates the reference framework)
    from stencilforge import analysis
    from stencilforge.frontend import bind_externals, inline_functions, parse_program

    meta = json.loads((GOLDEN / "corpus.json").read_text())
    assert len(meta) == 200
    for entry in meta[:60]:
        st = inline_functions(parse_program(entry["source"]))[0]
        impl = analysis.lower(bind_externals(st, {}))
        arrays = _inputs.random_field_arrays(impl, tuple(entry["domain"]),
                                             np.random.default_rng(entry["seed"]))
        for name, (arr, _) in arrays.items():
            assert _inputs.sha(arr) == entry["input_sha"][name], (entry["name"], name)
        scal = _inputs.random_scalars(impl, np.random.default_rng(entry["seed"] + 1))
        assert scal == entry["scalars"]


def test_reference_ref_kernels_present_or_skipped():
    """oracle/_ref holds the reference gen engine's own C kernels (built by
    oracle/build_ref.py in the build container)."""
    man = oracle.HERE / "_ref" / "manifest.json"
    if not man.exists():
        pytest.skip("oracle/_ref not built here")
    m = json.loads(man.read_text())
    assert set(m) == {"hdiff_f64", "hdiff_f32", "vadv_f64", "vadv_f32", "dycore_f64"}


def test_reference_ref_kernels_match_goldens(golden):
    """The reference's own kernels (the full-size checker of bench.py and the
    GPU tests) reproduce the golden vectors of its vec / debug engines."""
    if not oracle.ref_available("hdiff_f64"):
        pytest.skip("oracle/_ref not built here")
    for key in _cases(golden, "hdiff_"):
        got = oracle.ref_hdiff(golden[key + "_inp"], 0.05)
        assert np.array_equal(got, golden[key + "_out"]), key
    for key in _cases(golden, "vadv_"):
        got = oracle.ref_vadv(*(golden[f"{key}_{n}"] for n in "abcd"))
        assert np.array_equal(got, golden[key + "_x"]), key
    from paper_2311_08322_b200 import workloads

    g, keys = _dycore_cases()
    for key in keys:
        dom = tuple(int(x) for x in key.split("_")[1].split("x"))
        u, a, b, c = (workloads.dycore_arrays(dom, int(g[key + "_seed"]))[n] for n in "uabc")
        for s in range(int(g[key + "_steps"])):
            got = oracle.ref_dycore_run(u, a, b, c, s + 1)[2:-2, 2:-2, :]
            assert np.array_equal(got, g[f"{key}_out{s}"]), (key, s)


def _dycore_cases():
    g = np.load(GOLDEN / "dycore.npz")
    keys = sorted({k.rsplit("_", 1)[0] for k in g.files})
    return g, keys


def test_dycore_oracle_matches_reference_engines_bitwise():
    """oracle.dycore_run (C hdiff + C Thomas + numpy update) vs the
    reference's vec/debug engines running kernels/dycore.gts with the host
    swap (tests/golden/make_golden_dycore.py)."""
    from paper_2311_08322_b200 import workloads

    g, keys = _dycore_cases()
    assert keys
    for key in keys:
        dom = tuple(int(x) for x in key.split("_")[1].split("x"))
        u, a, b, c = (workloads.dycore_arrays(dom, int(g[key + "_seed"]))[n] for n in "uabc")
        state = u.copy()
        for s in range(int(g[key + "_steps"])):
            state[2:-2, 2:-2, :] = oracle.dycore_step(state, a, b, c, 0.05, 0.2)
            assert np.array_equal(state[2:-2, 2:-2, :], g[f"{key}_out{s}"]), (key, s)
