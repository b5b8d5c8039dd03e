"""Per-CUDA-source-line totals (instructions executed, warp stall samples) of an ncu report."""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None; inst = collections.Counter(); samp = collections.Counter(); src = {}
line = None
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    if r[0].strip():
        line = int(r[0]); src[line] = r[1][:90]
    try:
        inst[line] += float(r[hdr.index("Instructions Executed")] or 0)
        samp[line] += float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        pass
ti = sum(inst.values()); ts = sum(samp.values())
print(f"total inst {ti:.4g}  samples {ts:.4g}")
for l, v in sorted(inst.items(), key=lambda x: -x[1])[:top]:
    print(f"{l:5d} inst {100*v/ti:5.1f}%  stall {100*samp[l]/ts:5.1f}%  {src.get(l,'')}")
