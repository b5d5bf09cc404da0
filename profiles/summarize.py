"""Turn the round's ncu captures into committed summaries (runs here, no GPU).

    python profiles/summarize.py r1

Writes profiles/ncu_<round>.md (key metrics + top stalls per captured kernel,
launch-list shares) and profiles/ncu_traffic.json (DRAM bytes per launch, read
+ write; bench.py reports them as roofline.traffic).  The traffic comes from
the range-replay captures of tools/ncu_traffic.py (the launch followed by a
read-only L2 eviction, so the write-back is counted) when present, else from
the --set full captures (cold reads, but the writes still in L2 are missed).
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE.parent / "gpurun_out"
sys.path.insert(0, str(HERE))
from ncu_summary import KEYS  # noqa: E402

CAPTURES = {"vadv": "vadv_{r}", "hdiff": "hdiff64_{r}", "hdiff32": "hdiff32_{r}", "dycore": "dycore_{r}"}


def raw(path):
    txt = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return rows[0], rows[1], rows[2:]


def range_traffic(wl):
    """Read + write DRAM bytes of one launch from tools/ncu_traffic.py's
    range replay (launch + read-only eviction; reads minus the eviction)."""
    c, j = OUT / f"traffic_{wl}.csv", OUT / f"traffic_{wl}.json"
    if not (c.exists() and j.exists()):
        return None
    rows = [x for x in csv.reader(io.StringIO(c.read_text())) if len(x) > 12 and x[0] != "ID"]
    m = {x[10]: float(x[12].replace(",", "")) for x in rows}
    if "dram__bytes_read.sum" not in m:
        return None
    meta = json.loads([ln for ln in j.read_text().splitlines() if ln.startswith("{")][0])
    rd = m["dram__bytes_read.sum"] - meta["evict_read_bytes"]
    wr = m["dram__bytes_write.sum"]
    return {"dram_read_mb": rd / 1e6, "dram_write_mb": wr / 1e6, "traffic_bytes": rd + wr,
            "algorithmic_bytes": meta["algorithmic_bytes"],
            "traffic_over_algorithmic": round((rd + wr) / meta["algorithmic_bytes"], 3),
            "source": f"traffic_{wl}.csv: ncu --replay-mode range over [launch, gts_b200_l2_evict_read] "
                      f"(tools/ncu_traffic.py); reads minus the eviction's {meta['evict_read_bytes']} B"}


def main(r):
    md = [f"# ncu summaries, round {r}", "",
          "Captured on one B200 with `profiles/capture.sh " + r + "` (ncu --set full, --clock-control none,",
          "caches flushed between replays, so DRAM bytes are cold-cache per launch).  The traffic lines come",
          "from the range replays of tools/ncu_traffic.py, which include the write-back.", ""]
    traffic = {}
    for wl, pat in CAPTURES.items():
        rep = OUT / (pat.format(r=r) + ".ncu-rep")
        if not rep.exists():
            continue
        hdr, units, data = raw(rep)
        row = data[0]
        name = row[hdr.index("Kernel Name")]
        md += [f"## {wl}: `{name[:100]}`", "", "| metric | value | unit |", "|---|---|---|"]
        vals = {}
        for k in KEYS:
            if k in hdr:
                vals[k] = row[hdr.index(k)]
                md.append(f"| {k} | {vals[k]} | {units[hdr.index(k)]} |")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    stalls.append((float(row[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        md += ["", "top stall reasons (pc samples): " + ", ".join(f"{n} {int(v)}" for v, n in sorted(stalls, reverse=True)[:6]), ""]

        def mb(k):
            u = units[hdr.index(k)]
            v = float(row[hdr.index(k)])
            return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[u]

        rd, wr = mb("dram__bytes_read.sum"), mb("dram__bytes_write.sum")
        traffic[wl] = {"dram_read_mb": rd, "dram_write_mb": wr, "traffic_bytes": (rd + wr) * 1e6,
                       "duration_us": float(row[hdr.index("gpu__time_duration.sum")]),
                       "source": rep.name + " (kernel replay: writes still in L2 not counted)"}
        rr = range_traffic(wl)
        if rr is not None:
            traffic[wl] = rr
        t = traffic[wl]
        md += [f"DRAM traffic per launch incl. write-back: read {t['dram_read_mb']:.1f} MB + write "
               f"{t['dram_write_mb']:.1f} MB = {t['traffic_bytes'] / 1e6:.1f} MB"
               + (f" ({t['traffic_over_algorithmic']:.3f}x the algorithmic {t['algorithmic_bytes'] / 1e6:.1f} MB)"
                  if "algorithmic_bytes" in t else ""), ""]
    lst = OUT / f"launches_{r}.csv"
    if lst.exists():
        lines = [ln for ln in lst.read_text().splitlines() if ln.startswith('"')]
        rows = list(csv.reader(io.StringIO("\n".join(lines))))
        hdr = rows[0]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        agg = {}
        for rw in rows[1:]:
            n = rw[ki].split("(")[0]
            agg.setdefault(n, []).append(float(rw[vi].replace(",", "")))
        tot = sum(sum(v) for v in agg.values())
        md += ["## launch list (bench.py --steps 20, serialized under ncu)", "",
               "| kernel | launches | mean time | share |", "|---|---|---|---|"]
        for n, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            md.append(f"| {n} | {len(v)} | {sum(v) / len(v):.0f} {'ns'} | {sum(v) / tot:.1%} |")
    (HERE / f"ncu_{r}.md").write_text("\n".join(md) + "\n")
    (HERE / "ncu_traffic.json").write_text(json.dumps(traffic, indent=2) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
