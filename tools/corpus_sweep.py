"""Criterion-1 sweep over ALL 200 corpus programs on the GPU (evidence run).

    python tools/corpus_sweep.py [N] > gpurun_out/corpus_sweep.json

Compiles every program with a process pool (nvcc on the box, cache under
/tmp so the repo snapshot stays small), then runs each one on cuda:0 with
the reference harness inputs (tests/_inputs.py restatement of
corpus.random_field_args) and compares SHA-256 of every output compute view
with the reference debug engine's (tests/golden/corpus.json).  Also runs
each program through three launch configurations (default, no fusion, no
TMEM) to cover every lowering path, and (``tiles``) at the two tile-crossing
domains of tests/golden/corpus_tiles.json -- (37, 300, 9) and (70, 260, 120),
several fused / column tiles in i and j -- against the reference vec
engine's output hashes.
"""
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))
CACHE = "/tmp/gts_corpus_cache"
OPTS = [None, {"fuse_parallel": False}, {"tmem": False, "tma": False}]


def _compile(args):
    idx, src, name, oi = args
    import paper_2311_08322_b200 as b200

    t0 = time.time()
    try:
        st = b200.compile_stencil(src, name, cache_dir=CACHE, gen_options=OPTS[oi])
        return idx, oi, st.build_info["plan"], None, time.time() - t0
    except Exception as exc:  # reported
        return idx, oi, None, f"{type(exc).__name__}: {exc}"[:300], time.time() - t0


def _compile_default(args):
    src, name = args
    import paper_2311_08322_b200 as b200

    b200.compile_stencil(src, name)
    return name


def prebuild(sources, names) -> None:
    """nvcc modules into the default (in-tree) cache with a process pool."""
    with ProcessPoolExecutor(max_workers=min(16, os.cpu_count() or 8)) as ex:
        list(ex.map(_compile_default, list(zip(sources, names))))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    print(json.dumps(sweep(n), indent=1))


def _run_one(b200, _inputs, np, st, dom, seed, scalars, outputs, want_sha) -> str:
    arrays = _inputs.random_field_arrays(st.implementation, dom, np.random.default_rng(seed))
    fields = {k: b200.from_array(a, o) for k, (a, o) in arrays.items()}
    st(domain=dom, **fields, **scalars)
    ok = all(_inputs.sha(_inputs.compute_view(fields[o].host_array(), fields[o].origin, dom))
             == want_sha[o] for o in outputs)
    return "bitwise" if ok else "MISMATCH"


def sweep(n: int = 200, configs=None, tiles: bool = True) -> dict:
    meta = json.loads((REPO / "tests" / "golden" / "corpus.json").read_text())[:n]
    tile_meta = json.loads((REPO / "tests" / "golden" / "corpus_tiles.json").read_text())[:n] if tiles else []
    cfgs = range(len(OPTS)) if configs is None else configs
    jobs = [(e["idx"], e["source"], e["name"], oi) for e in meta for oi in cfgs]
    t0 = time.time()
    with ProcessPoolExecutor(max_workers=os.cpu_count() or 8) as ex:
        comp = {(i, oi): (plan, err) for i, oi, plan, err, _ in ex.map(_compile, jobs)}
    t_comp = time.time() - t0
    import numpy as np
    import _inputs
    import paper_2311_08322_b200 as b200

    results, kinds = [], {}
    for e in meta:
        for oi in cfgs:
            plan, err = comp[(e["idx"], oi)]
            rec = {"idx": e["idx"], "opts": OPTS[oi], "plan": plan}
            if err:
                rec["status"] = "compile_error"
                rec["error"] = err
                results.append(rec)
                continue
            st = b200.compile_stencil(e["source"], e["name"], cache_dir=CACHE, gen_options=OPTS[oi])
            runs = [(tuple(e["domain"]), e["seed"], e["scalars"], e["output_sha"])]
            if tiles:
                tm = tile_meta[e["idx"]]
                assert tm["name"] == e["name"]
                runs += [(tuple(r["domain"]), r["seed"], r["scalars"], r["output_sha"]) for r in tm["runs"]]
            rec["domains"] = {}
            try:
                for dom, seed, scalars, want in runs:
                    rec["domains"][str(dom)] = _run_one(b200, _inputs, np, st, dom, seed, scalars,
                                                        e["outputs"], want)
                bad = [d for d, v in rec["domains"].items() if v != "bitwise"]
                rec["status"] = "MISMATCH" if bad else "bitwise"
                if bad:
                    rec["mismatch_domains"] = bad
            except Exception as exc:
                rec["status"] = "run_error"
                rec["error"] = f"{type(exc).__name__}: {exc}"[:300]
            for k in plan:
                kinds[k.split(":")[0]] = kinds.get(k.split(":")[0], 0) + 1
            results.append(rec)
    summary = {"programs": len(meta), "configs": len(list(cfgs)), "compile_s": round(t_comp, 1),
               "domains_per_program": 1 + (2 if tiles else 0), "status": {}, "kernel_kinds": kinds}
    for r in results:
        summary["status"][r["status"]] = summary["status"].get(r["status"], 0) + 1
    return {"summary": summary, "failures": [r for r in results if r["status"] != "bitwise"]}


if __name__ == "__main__":
    main()
