"""The reference's CLI (stencilforge cli.py: gts run / diff / bench) with the
b200 backend registered by ``install()`` -- drop-in at the command line
(SURVEY.md 8(f)4)."""

import json

import numpy as np
import pytest

import oracle


def _cli():
    import paper_2311_08322_b200 as b200

    b200.install()
    from click.testing import CliRunner
    from stencilforge import cli

    return CliRunner(), cli.main


def _kernel_file(tmp_path, name):
    from stencilforge.kernels import kernel_source

    p = tmp_path / f"{name}.gts"
    p.write_text(kernel_source(name))
    return str(p)


def test_install_registers_backend_in_cli():
    import paper_2311_08322_b200 as b200

    b200.install()
    import stencilforge
    from stencilforge import backends, cli, runtime

    assert "b200" in backends.BACKEND_IDS and "b200" in runtime.BACKEND_IDS
    assert cli.compile_stencil is b200.compile_stencil
    assert stencilforge.compile_stencil is b200.compile_stencil


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["hdiff", "vadv"])
def test_cli_diff_b200_vs_vec(gpu, tmp_path, kernel):
    runner, main = _cli()
    f = _kernel_file(tmp_path, kernel)
    args = ["diff", f, "--backends", "vec,b200", "--sizes", "16,32:24:80", "--tol", "0"]
    if kernel == "vadv":
        for n, lo_hi in (("a", "0.1:0.45"), ("c", "0.1:0.45"), ("b", "1.0:2.0")):
            args += ["--range", f"{n}={lo_hi}"]
    res = runner.invoke(main, args)
    assert res.exit_code == 0, res.output
    lines = [json.loads(ln) for ln in res.output.splitlines() if ln.startswith("{")]
    assert lines and all(ln["max_rel"] == 0.0 for ln in lines)


@pytest.mark.gpu
def test_cli_run_gtsf_roundtrip(gpu, tmp_path):
    from stencilforge import storage

    runner, main = _cli()
    f = _kernel_file(tmp_path, "hdiff")
    rng = np.random.default_rng(5)
    vals = rng.uniform(-1, 1, (36, 28, 7))
    storage.write_gtsf(storage.from_array(vals, (2, 2, 0)), str(tmp_path / "inp.gtsf"))
    res = runner.invoke(main, ["run", f, "--backend", "b200", "--in", f"inp={tmp_path / 'inp.gtsf'}",
                               "--out", f"out={tmp_path / 'out.gtsf'}", "--scalar", "coeff=0.05"])
    assert res.exit_code == 0, res.output
    out = storage.read_gtsf(str(tmp_path / "out.gtsf"))
    assert np.array_equal(np.asarray(out.view), oracle.hdiff_c(vals, 0.05))


@pytest.mark.gpu
def test_cli_bench_b200(gpu):
    runner, main = _cli()
    res = runner.invoke(main, ["bench", "--kernels", "hdiff,vadv", "--backends", "b200",
                               "--sizes", "32", "--nk", "16", "--reps", "5"])
    assert res.exit_code == 0, res.output
    assert "b200" in res.output
