"""Per-source-line instruction and stall-sample shares of an ncu report, sorted by stall,
with dsea_force.cu line-range categories (approximate: the source page mixes files):
python scripts/ncu_lines_stall.py <report.ncu-rep> <top> [line_lo line_hi]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr=None; inst=collections.Counter(); samp=collections.Counter(); src={}; line=None
for r in rows:
    if len(r) > 3 and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < len(hdr): continue
    if r[0].strip(): line = int(r[0]); src[line] = r[1][:80]
    try:
        inst[line] += float(r[hdr.index("Instructions Executed")] or 0)
        samp[line] += float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError: pass
ti=sum(inst.values()); ts=sum(samp.values())
# category ranges (dsea_force.cu line numbers)
cats = {"table(99-216)":(99,216),"staging(265-318)":(265,318),"chunk-setup+bsearch(320-372)":(320,372),"pair(374-397)":(374,397),"flush(398-423)":(398,423),"screen(424-458)":(424,458),"integrate+energy(459-524)":(459,524)}
agg = collections.Counter(); aggs=collections.Counter()
for l in inst:
    for k,(a,b) in cats.items():
        if l is not None and a <= l <= b: agg[k]+=inst[l]; aggs[k]+=samp[l]
print("category shares (inst%, stall%) -- lines outside dsea_force.cu (device.cuh helpers) not attributed:")
for k in cats: print(f"  {k:32s} {100*agg[k]/ti:5.1f} {100*aggs[k]/ts:5.1f}")
print("top by stall:")
for l, v in sorted(samp.items(), key=lambda x: -x[1])[:top]:
    print(f"{l:5d} inst {100*inst[l]/ti:5.1f}%  stall {100*v/ts:5.1f}%  {src.get(l,'')}")
if len(sys.argv) > 4:
    a, b = int(sys.argv[3]), int(sys.argv[4])
    print(f"lines {a}-{b}:")
    for l in sorted(k for k in inst if k is not None and a <= k <= b):
        print(f"{l:5d} inst {100*inst[l]/ti:5.2f}%  stall {100*samp[l]/ts:5.2f}%  {src.get(l,'')}")
