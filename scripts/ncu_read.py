"""Summarise one ncu report: headline metrics, stall reasons, and the SASS regions
(runs of instructions with the same execution count) that carry the time.
usage: python scripts/ncu_read.py gpurun_out/<tag>.ncu-rep [min_pct]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
minp = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for r in rows[2:]:
    for w in want:
        if w in h:
            print(f"  {w} = {r[h.index(w)][:80]}")
    st = [(float(r[i] or 0), x.split("issue_stalled_")[1].split("_per_issue")[0]) for i, x in enumerate(h)
          if "issue_stalled" in x and "per_issue_active" in x]
    print("  stalls/issue:", " ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = [i for i, r in enumerate(rows) if "Address" in r][0]
h = rows[hi]
data = rows[hi + 1:]
ie, isamp, iw, isrc = h.index("Instructions Executed"), h.index("# Samples"), h.index("L1 Wavefronts Shared"), h.index("Source")
f = lambda r, i: int(r[i] or 0)
tot = sum(f(r, ie) for r in data) or 1
tots = sum(f(r, isamp) for r in data) or 1
print(f"  SASS lines {len(data)}, warp instructions {tot}, samples {tots}")
cur, start, acc, accs, accw = None, 0, 0, 0, 0
out = []
for i, r in enumerate(data):
    e = f(r, ie)
    if cur is None or abs(e - cur) > 0.03 * max(cur, 1) + 10:
        if cur is not None:
            out.append((start, i - 1, cur, acc, accs, accw))
        cur, start, acc, accs, accw = e, i, 0, 0, 0
    acc += e; accs += f(r, isamp); accw += f(r, iw)
out.append((start, len(data) - 1, cur, acc, accs, accw))
for s, e, c, a, sm, w in out:
    if 100 * a / tot >= minp or 100 * sm / tots >= minp:
        print(f"  [{s:5d}-{e:5d}] n={e-s+1:4d} exec={c:9d} instr%={100*a/tot:5.1f} samp%={100*sm/tots:5.1f} smem_wf={w}  {data[s][isrc][:50]}")
