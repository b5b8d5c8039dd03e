"""Summarise an ncu report: key metrics, stall reasons, hottest SASS blocks."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u = rows[0], rows[1]
for v in rows[2:]:
    d = dict(zip(h, v))
    print("kernel:", d.get("Kernel Name", "")[:80])
    keys = ["gpu__time_duration.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
            "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
            "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__occupancy_limit_shared_mem",
            "launch__occupancy_limit_registers"]
    for k in keys:
        if k in d:
            print(f"  {k:70s} {d[k]:>16s} {u[h.index(k)]}")
    st = [(k, float(d[k])) for k in h if k.startswith("smsp__average_warps_issue_stalled_")
          and k.endswith("_per_issue_active.ratio") and d[k] not in ("", "n/a")]
    print("  stalls (warps per issue):", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}"
                                                   for k, v in sorted(st, key=lambda x: -x[1])[:8]))
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(sass.splitlines()))
if len(rows) > 2:
    h = rows[1]; data = rows[2:]
    iS = h.index("Source"); iE = h.index("Instructions Executed"); iW = h.index("Warp Stall Sampling (All Samples)")
    E = [int(r[iE]) if r[iE].isdigit() else 0 for r in data]
    W = [int(r[iW]) if r[iW].isdigit() else 0 for r in data]
    blocks, start = [], 0
    for i in range(1, len(E) + 1):
        if i == len(E) or E[i] != E[start]:
            blocks.append((start, i - 1, E[start], sum(E[start:i]), sum(W[start:i])))
            start = i
    tot, ws = max(1, sum(E)), max(1, sum(W))
    print("  hottest SASS blocks (instr share / stall-sample share):")
    for b in sorted(blocks, key=lambda b: -(b[3] / tot + b[4] / ws))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
        print(f"   {b[0]:5d}-{b[1]:5d} x{b[2]:<9d} n={b[1]-b[0]+1:4d} inst={b[3]/tot*100:5.1f}% stall={b[4]/ws*100:5.1f}%  {data[b[0]][iS].strip()[:60]}")

# ---- per-region stall reasons (regions split at barriers / big count changes) ----
if len(sys.argv) > 3 and len(rows) > 2:
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    idx = {c: h.index(c) for c in reasons}
    regs = [(int(a), int(b), n) for a, b, n in (x.split(":") for x in sys.argv[3].split(","))]
    tot = {c: sum(int(r[idx[c]]) for r in data if r[idx[c]].isdigit()) for c in reasons}
    allt = sum(tot.values())
    for a, b, n in regs:
        sub = {c: sum(int(r[idx[c]]) for r in data[a:b] if r[idx[c]].isdigit()) for c in reasons}
        s = sum(sub.values())
        top = sorted(sub.items(), key=lambda x: -x[1])[:5]
        print(f"  {n:14s} {s/allt*100:5.1f}% of samples: " + ", ".join(f"{k[6:]}={v/allt*100:.1f}%" for k, v in top))
