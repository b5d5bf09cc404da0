"""Golden hashes of the 200-program corpus at TILE-CROSSING domains, produced
by running the REFERENCE's own ``vec`` engine (build container only):

    python tests/golden/make_golden_tiles.py

The reference's criterion-1 corpus (corpus.generate_corpus(seed=2024),
test_acceptance.py:34-35, 116-129) runs at CORPUS_DOMAINS (at most 16 points
per axis).  The b200 templates tile the horizontal plane (fused PARALLEL
tiles of 4/8/16 rows x 128 columns, column tiles of 8 rows x 32 columns), so
the cross-tile hazard rules of the lowering (lowering._fuse_parallel) are
only exercised by domains that span several tiles in both i and j.  This
script runs every program at

  * (37, 300, 9)    -- < 2 M points: the tiny-domain fused geometry (4-row tiles);
  * (70, 260, 120)  -- >= 2 M points: the default fused geometry (8-row tiles);

with the corpus harness inputs (tests/_inputs.py restatement of
corpus.random_field_args, pinned here against the reference for every
program's first domain) and stores the SHA-256 of every output compute view
in ``corpus_tiles.json``.  ``vec`` and ``debug`` agree bitwise on this corpus
(criterion 1; make_golden.py asserts it at CORPUS_DOMAINS); ``debug`` is too
slow for 2 M points.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("GTS_CACHE_DIR", tempfile.mkdtemp(prefix="gts-golden-"))

import stencilforge as sf  # noqa: E402
from stencilforge import corpus  # noqa: E402

import _inputs  # noqa: E402

TILE_DOMAINS = [(37, 300, 9), (70, 260, 120)]
CORPUS_N = 200


def main() -> None:
    progs = corpus.generate_corpus(seed=2024, count=CORPUS_N)
    meta = json.loads((HERE / "corpus.json").read_text())
    out = []
    t0 = time.time()
    for idx, p in enumerate(progs):
        assert meta[idx]["name"] == p.name and meta[idx]["source"] == p.source
        stv = sf.compile_stencil(p.source, p.name, backend="vec")
        impl = stv.implementation
        lay = sf.default_layout("vec")
        runs = []
        for di, dom in enumerate(TILE_DOMAINS):
            seed = 70_000 + 10 * idx + di
            arrays = _inputs.random_field_arrays(impl, dom, np.random.default_rng(seed))
            scalars = _inputs.random_scalars(impl, np.random.default_rng(seed + 1))
            if di == 0:  # pin the restatement against the reference harness builder
                ref = corpus.random_field_args(impl, "vec", dom, np.random.default_rng(seed))
                for f in impl.api_fields:
                    assert np.array_equal(np.asarray(ref[f.name].data()), arrays[f.name][0], equal_nan=True)
                assert corpus.random_scalar_args(impl, np.random.default_rng(seed + 1)) == scalars
            fields = {n: sf.from_array(a, o, lay) for n, (a, o) in arrays.items()}
            stv(domain=dom, **fields, **scalars)
            runs.append({
                "domain": list(dom), "seed": seed, "scalars": scalars,
                "output_sha": {o: _inputs.sha(np.asarray(fields[o].compute_view(dom)))
                               for o in p.outputs},
            })
        out.append({"idx": idx, "name": p.name, "runs": runs})
        if idx % 20 == 0:
            print(f"{idx} programs, {time.time() - t0:.0f} s", file=sys.stderr)
    (HERE / "corpus_tiles.json").write_text(json.dumps(out, indent=0))
    print("corpus_tiles.json", (HERE / "corpus_tiles.json").stat().st_size)


if __name__ == "__main__":
    main()
