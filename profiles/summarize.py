"""Turn one round's raw GPU captures (gpurun_out/) into the committed profiles/.

    python profiles/summarize.py <prefix> <round>

Inputs (written by gpurun):
  gpurun_out/<prefix>_bench.json     python bench.py (the driver's default line)
  gpurun_out/<prefix>_launches.csv   ncu --metrics gpu__time_duration.sum --csv launch list
  gpurun_out/<prefix>_full_raw.csv   its raw page (METRICS), converted on the box
                                     (or gpurun_out/<prefix>_full.ncu-rep itself)
Outputs:
  profiles/r<round>_bench_c2.json, r<round>_launches.csv, r<round>_ncu_summary.txt,
  traffic.json (dram bytes per launch of the dominant kernel families, read by bench.py)
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
]
SHORT = ["ms", "dram_rd_GB", "dram_wr_GB", "regs", "grid", "block", "warps_active%", "issue%",
         "alu_pipe%", "fma_pipe%", "l1_data_pipe%", "smem_wavefronts", "smem_conflicts", "dram%",
         "warp_instr"]


def family(name: str) -> str:
    return name.replace("void ", "").replace("qmsort_b200::", "").split("<")[0].split("(")[0]


def to_us(unit: str, v: float) -> float:
    return {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3,
            "msecond": v * 1e3}[unit]


def main() -> None:
    prefix, rnd = sys.argv[1], sys.argv[2]
    line = open(os.path.join(G, f"{prefix}_bench.json")).read().strip().splitlines()[-1]
    bench = json.loads(line)
    json.dump(bench, open(os.path.join(P, f"r{rnd}_bench_c2.json"), "w"), indent=1)

    # launch list: every launch, and the family shares of the last whole sort
    rows = list(csv.reader(open(os.path.join(G, f"{prefix}_launches.csv"))))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                out.append((int(d["ID"]), d["Kernel Name"].split("(")[0][:90],
                            to_us(d["Metric Unit"], float(d["Metric Value"].replace(",", "")))))
    start = max(i for i, o in enumerate(out) if "init_level_kernel" in o[1])
    sort_l = out[start:]
    tot = sum(u for _, _, u in sort_l)
    fam: dict = {}
    for _, k, u in sort_l:
        fam[family(k)] = fam.get(family(k), 0.0) + u
    with open(os.path.join(P, f"r{rnd}_launches.csv"), "w") as fh:
        fh.write("# ncu launch list (gpu__time_duration.sum, --clock-control none), "
                 "python bench.py --steps 1 --warmup 1 --quick\n")
        fh.write("# cold-cache, serialised per-launch times: compare shares, not absolutes.\n")
        fh.write("# last whole sort (from the last init_level_kernel): "
                 + ", ".join(f"{k} {v:.0f} us ({v / tot:.1%})" for k, v in fam.items())
                 + f"; total {tot:.0f} us over {len(sort_l)} launches\n")
        fh.write("id,kernel,us\n")
        for i, k, u in out:
            fh.write(f"{i},{k},{u:.1f}\n")

    # full capture: one row per launch
    rawcsv = os.path.join(G, f"{prefix}_full_raw.csv")  # converted on the GPU box (scripts/gpu_profile.sh)
    if os.path.exists(rawcsv):
        raw = open(rawcsv).read()
    else:
        rep = os.path.join(G, f"{prefix}_full.ncu-rep")
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                             capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h = r[0]
    lines = [f"# ncu --set full --clock-control none, bench.py --quick (C2 2^28 uint32), round {rnd}",
             "# kernel | " + " | ".join(SHORT)]
    traffic: dict = {}
    for row in r[2:]:
        d = dict(zip(h, row))
        vals = []
        for m in METRICS:
            v = d.get(m, "")
            try:
                f = float(v.replace(",", ""))
                vals.append(f"{f:.4g}")
            except ValueError:
                vals.append(v)
        name = family(d["Kernel Name"]) + ("<" + d["Kernel Name"].split("<")[1].split(">")[0] + ">"
                                           if "<" in d["Kernel Name"] else "")
        lines.append(f"{name} | " + " | ".join(vals))
        f = family(d["Kernel Name"]).replace("_kernel", "").replace("blocksort_tasks", "blocksort").replace("tablesort_tasks", "blocksort")
        try:
            b = (float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])) * 1e9
        except ValueError:
            continue
        traffic.setdefault(f, []).append(b)
    with open(os.path.join(P, f"r{rnd}_ncu_summary.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    # per launch, averaged over the captured launches of the family (blocksort:
    # per sort, i.e. summed over its size-class launches of one sort)
    tj = {}
    if "scatter" in traffic:
        tj["scatter"] = sum(traffic["scatter"]) / len(traffic["scatter"])
    if "count" in traffic:
        tj["count"] = sum(traffic["count"]) / len(traffic["count"])
    if "blocksort" in traffic:
        nsorts = max(1, len([x for x in traffic.get("scatter", [])]) // 2)
        tj["blocksort"] = sum(traffic["blocksort"]) / nsorts
    tj["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum from "
                   f"profiles/r{rnd}_ncu_summary.txt; scatter/count per launch, blocksort per sort")
    json.dump(tj, open(os.path.join(P, "traffic.json"), "w"), indent=1)
    print(json.dumps({k: (v / tot) for k, v in fam.items()}), tot)


def configs(prefix: str, rnd: str) -> None:
    """The other configs' bench lines (scripts/gpu_profile.sh: cfg_*, merge_*, sharded_*)
    condensed into profiles/r<round>_configs.json."""
    out = {}
    for f in sorted(os.listdir(G)):
        if not (f.startswith(prefix + "_") and f.endswith(".json")):
            continue
        tag = f[len(prefix) + 1:-5]
        if not tag.startswith(("cfg_", "merge_", "sharded_")):
            continue
        try:
            d = json.loads(open(os.path.join(G, f)).read().strip().splitlines()[-1])
        except (ValueError, IndexError):
            continue
        e = {k: d[k] for k in ("value", "unit", "ms_per_step", "config") if k in d}
        if "sort_roofline" in d:
            e["sort_roofline_frac"] = d["sort_roofline"]["frac"]
            e["phases_us"] = {k: v["us"] for k, v in d["sort_roofline"]["phases"].items()}
            r = d.get("roofline", {})
            e["dominant"] = {k: r.get(k) for k in ("kernel", "achieved", "frac", "avg_launch_us")}
        else:
            for k in ("verify", "roofline"):
                if k in d:
                    e[k] = d[k]
        out[tag] = e
    if out:
        json.dump(out, open(os.path.join(P, f"r{rnd}_configs.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
    configs(sys.argv[1], sys.argv[2])
