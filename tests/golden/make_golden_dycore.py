"""Golden fixtures for the dycore step (BASELINE.json configs[4]) produced by
the REFERENCE engines themselves.  Build container only (needs /root/reference):

    python tests/golden/make_golden_dycore.py

The program is paper_2311_08322_b200/kernels/dycore.gts (authored in the
reference DSL; the reference ships no dycore stencil).  For
each case the reference ``vec`` engine (and ``debug`` for the small case)
runs ``steps`` time steps with the host swap u_out -> u_in; the initial state
and every step's u_out compute view are stored in dycore.npz.
"""

from __future__ import annotations

import os
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("GTS_CACHE_DIR", tempfile.mkdtemp(prefix="gts-golden-"))

import stencilforge as sf  # noqa: E402

SRC = (REPO / "paper_2311_08322_b200" / "kernels" / "dycore.gts").read_text()
COEFF, TAU = 0.05, 0.2
CASES = [((10, 12, 6), 3, 11, ("debug", "vec")), ((24, 20, 16), 3, 12, ("vec",)),
         ((16, 40, 80), 2, 13, ("vec",))]


def gen(domain, seed):
    # same generator as paper_2311_08322_b200.workloads.dycore_arrays
    ni, nj, nk = domain
    rng = np.random.default_rng(seed)
    u = rng.uniform(-1.0, 1.0, (ni + 4, nj + 4, nk))
    a = -rng.uniform(0.0, 0.5, (ni, nj, nk))
    c = -rng.uniform(0.0, 0.5, (ni, nj, nk))
    return u, a, 1.0 - a - c, c


def run(backend, domain, steps, u, a, b, c):
    st = sf.compile_stencil(SRC, "dycore", backend=backend)
    lay = sf.default_layout(backend)
    bufs = [sf.from_array(u, (2, 2, 0), lay), sf.from_array(u, (2, 2, 0), lay)]
    fa = {n: sf.from_array(v, (0, 0, 0), lay) for n, v in (("a", a), ("b", b), ("c", c))}
    outs = []
    for s in range(steps):
        src, dst = bufs[s % 2], bufs[(s + 1) % 2]
        st(u_in=src, u_out=dst, coeff=COEFF, tau=TAU, **fa)
        outs.append(np.asarray(dst.data())[2:-2, 2:-2, :].copy())
    return outs


def main():
    out = {}
    for domain, steps, seed, engines in CASES:
        u, a, b, c = gen(domain, seed)
        key = "dycore_%dx%dx%d" % domain
        res = {e: run(e, domain, steps, u, a, b, c) for e in engines}
        for e in engines[1:]:
            for x, y in zip(res[engines[0]], res[e]):
                assert np.array_equal(x, y), f"{e} != {engines[0]}"
        out[key + "_seed"] = np.array(seed)
        out[key + "_steps"] = np.array(steps)
        for s, v in enumerate(res[engines[-1]]):
            out[f"{key}_out{s}"] = v
        print(key, "steps", steps, "engines", engines, "max |u|", float(np.abs(res[engines[-1]][-1]).max()))
    np.savez_compressed(HERE / "dycore.npz", **out)


if __name__ == "__main__":
    main()
