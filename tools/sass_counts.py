#!/usr/bin/env python
"""Per-kernel SASS evidence of the shipped modules.

    python tools/sass_counts.py > profiles/sass_r2.txt

Runs ``cuobjdump -sass`` on the prebuilt benchmark modules (the in-tree
module cache) and counts, per kernel, the instructions that prove the
Blackwell paths (TMA loads / L2 prefetches / stores UTMALDG / UTMAPF / UTMASTG, Tensor Memory
STTM / LDTM, mbarrier SYNCS.*), the FP64 arithmetic (DADD, DMUL, DFMA: the
parity build has no contraction, so DFMA appears only in the exact-replay
division of gts_common.cuh), and the XU-pipe conversions (F2F) and MUFU.
"""
import re
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2311_08322_b200 as b200  # noqa: E402
from paper_2311_08322_b200 import workloads  # noqa: E402

OPS = ["UTMALDG", "UTMAPF", "UTMASTG", "UBLKCP", "STTM", "LDTM", "SYNCS", "DADD", "DMUL", "DFMA", "F2F", "MUFU",
       "LDS", "STS", "STG", "LDG", "SHFL"]
MODULES = [("hdiff", "f64", None), ("hdiff", "f32", None), ("vadv", "f64", None), ("vadv", "f32", None),
           ("dycore", "f64", None), ("dycore", "f64", {"mirror": "u_out"})]


def counts(so: str) -> dict:
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
    out = {}
    for chunk in re.split(r"\n\s+Function : ", sass)[1:]:
        name = chunk.split("\n", 1)[0].strip()
        ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)(?:\.[A-Z0-9_.]+)?", chunk)
        c = {k: sum(1 for o in ops if o == k) for k in OPS}
        c["total"] = len(ops)
        out[name] = c
    return out


def main():
    print("# SASS instruction counts of the shipped modules (cuobjdump -sass; tools/sass_counts.py)\n")
    print("| module | kernel | " + " | ".join(OPS) + " | total |")
    print("|---|---|" + "---|" * (len(OPS) + 1))
    for kernel, dtype, opts in MODULES:
        st = b200.compile_stencil(workloads.source(kernel, dtype), kernel, gen_options=opts)
        so = st.build_info["so_path"]
        tag = f"{kernel} {dtype}" + (f" {opts}" if opts else "")
        for fn, c in counts(so).items():
            if "fill_nan" in fn:
                continue
            short = re.sub(r"^_Z\d+", "", fn).split("9GtsParams")[0]
            print(f"| {tag} | {short} | " + " | ".join(str(c[k]) for k in OPS) + f" | {c['total']} |")
    lib = Path(b200.__file__).resolve().parent / "libgts_b200.so"
    for fn, c in counts(str(lib)).items():
        short = re.sub(r"^_Z\d+", "", fn)[:40]
        print(f"| libgts_b200 | {short} | " + " | ".join(str(c[k]) for k in OPS) + f" | {c['total']} |")


if __name__ == "__main__":
    main()
