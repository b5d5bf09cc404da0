"""Build oracle/_ref: the REFERENCE's own native kernels for hdiff / vadv
(and the dycore step).

TEST / BASELINE INFRASTRUCTURE ONLY (never linked by the product).

The reference's only native code is the C translation unit its ``gen``
engine emits per stencil (stencilforge ``backends/gen.py:229-369``).  This
script runs that emitter from the read-only reference tree (build container
only), writes the generated C into ``oracle/_ref/`` and compiles it with the
reference's own flags (``gen.py:64-67``: ``-O3 -fPIC -shared -fopenmp
-ffp-contract=off``).  ``oracle/_ref`` is git-ignored but travels to the GPU
box with the snapshot, where ``bench.py --impl reference`` times it on the
host cores and the GPU parity tests use it as a second oracle.

    python oracle/build_ref.py
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "_ref"
REF_SRC = Path("/root/reference/pkg/src")

KERNELS = {
    # key: (kernel name, dtype substitution)
    "hdiff_f64": ("hdiff", None),
    "hdiff_f32": ("hdiff", "f32"),
    "vadv_f64": ("vadv", None),
    "vadv_f32": ("vadv", "f32"),
    # BASELINE configs[4]: the dycore step, authored in the reference DSL
    # (paper_2311_08322_b200/kernels/dycore.gts; the reference ships no
    # dycore) and compiled by the reference's own gen emitter -- the
    # full-size multi-step parity checker
    "dycore_f64": ("dycore", None),
}
DYCORE_GTS = HERE.parent / "paper_2311_08322_b200" / "kernels" / "dycore.gts"


def main() -> int:
    if not (REF_SRC / "stencilforge").is_dir():
        print("reference tree not present; oracle/_ref not rebuilt", file=sys.stderr)
        return 0
    sys.path.insert(0, str(REF_SRC))
    os.environ.setdefault("GTS_CACHE_DIR", tempfile.mkdtemp(prefix="gts-ref-"))
    from stencilforge import analysis, ir
    from stencilforge.backends import gen
    from stencilforge.frontend import bind_externals, inline_functions, parse_program
    from stencilforge.kernels import kernel_source

    OUT.mkdir(exist_ok=True)
    manifest = {}
    env = dict(os.environ)
    env.pop("CC", None)
    for key, (name, dt) in KERNELS.items():
        src = DYCORE_GTS.read_text() if name == "dycore" else kernel_source(name)
        if dt:
            src = src.replace("Field[f64]", f"Field[{dt}]")
        items = inline_functions(parse_program(src))
        bound = bind_externals(items[0], {})
        impl = analysis.lower(bound)
        fp = ir.fingerprint(bound, "gen", {}, gen.toolchain_version(), None)
        c_src = gen.generate_source(impl, fp)
        c_path = OUT / f"{key}.c"
        so_path = OUT / f"lib{key}.so"
        c_path.write_text(c_src)
        cmd = ["cc", "-O3", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
               str(c_path), "-o", str(so_path), "-lm"]
        subprocess.run(cmd, check=True, env=env)
        manifest[key] = {
            "so": so_path.name,
            "symbol": gen.entry_name(impl, fp),
            "fields": [f.name for f in impl.api_fields],
            "scalars": [[s.name, s.dtype] for s in impl.api_scalars],
            "dtype": dt or "f64",
            "flags": "-O3 -fPIC -shared -fopenmp -ffp-contract=off",
            "emitter": "stencilforge/backends/gen.py:229-369",
        }
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=2))
    print(f"built {len(manifest)} reference kernels into {OUT}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
