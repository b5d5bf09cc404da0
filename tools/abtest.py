"""Interleaved A/B timing of gen_options variants (median of R alternating
rounds; each round = bench-style graph replay of 200 launches over rotating
input sets), to separate small effects from run-to-run drift:

    python tools/abtest.py hdiff f64 256x256x80 5 '{}' '{"pf_swz": true}'
"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import ksweep  # noqa: E402

kernel, dtype, dom_s, rounds = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
dom = tuple(int(x) for x in dom_s.split("x"))
opts = [json.loads(o) for o in sys.argv[5:]]
res = {i: [] for i in range(len(opts))}
for _ in range(rounds):
    for i, o in enumerate(opts):
        us, _, _ = ksweep.time_one(kernel, dtype, dom, o)
        res[i].append(us)
for i, o in enumerate(opts):
    print(f"{kernel} {dtype} {dom_s} {json.dumps(o)}: median {statistics.median(res[i]):.2f} us "
          f"(min {min(res[i]):.2f}, max {max(res[i]):.2f}, n={rounds})", flush=True)
