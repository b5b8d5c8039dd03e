"""Shared-memory wavefronts (and excess from bank conflicts) and stall samples per CUDA
source line of an ncu report: python scripts/ncu_smem.py <report> [top]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
wf = collections.Counter(); ex = collections.Counter(); st = collections.Counter(); src = {}
hdr = None; line = None
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < len(hdr) - 5:
        continue
    if r[0] and r[1]:          # CUDA source line row
        line = int(r[0]) if r[0].isdigit() else None
        if line is not None: src[line] = r[1][:90]
        continue
    d = dict(zip(hdr[2:], r[2:])) if False else None
for r in rows:
    pass
# second pass: SASS rows carry the metrics; the CUDA line they belong to precedes them
line = None
iw = hdr.index("L1 Wavefronts Shared"); ie = hdr.index("L1 Wavefronts Shared Excessive")
iss = hdr.index("Warp Stall Sampling (All Samples)")
for r in rows:
    if len(r) != len(hdr) or r[0] == "Line No":
        continue
    if r[0].strip():
        line = int(r[0]) if r[0].strip().isdigit() else None
    if line is None: continue
    def num(x):
        try: return float(x)
        except: return 0.0
    wf[line] += num(r[iw]); ex[line] += num(r[ie]); st[line] += num(r[iss])
tw = sum(wf.values()); te = sum(ex.values()); ts = sum(st.values())
print(f"smem wavefronts {tw:.3e}, excessive {te:.3e}; stall samples {ts:.3e}")
for l, w in wf.most_common(top):
    print(f"{l:5d} wf {100*w/tw:5.1f}%  excess {100*ex[l]/max(w,1):5.1f}%  stall {100*st[l]/ts:5.1f}%  {src.get(l,'')}")
