"""Summarise DSEA_TIMELINE CSVs (one per rank): compute-stream busy time, idle gaps,
first start (pipeline fill), end, and copy-engine hop time."""
import csv
import glob
import sys

for prefix in sys.argv[1:]:
    files = sorted(glob.glob(prefix + ".rank*.csv"))
    print(prefix)
    for f in files:
        rows = [(r["kind"], float(r["start_ms"]), float(r["end_ms"])) for r in csv.DictReader(open(f))]
        cs = sorted((a, b, k) for k, a, b in rows if k in ("force", "bin"))
        hop = sum(b - a for k, a, b in rows if k == "hop")
        busy = sum(b - a for a, b, _ in cs)
        force = sum(b - a for a, b, k in cs if k == "force")
        gaps = [cs[i + 1][0] - cs[i][1] for i in range(len(cs) - 1)]
        big = sorted(gaps)[-5:]
        gf = [cs[i + 1][0] - cs[i][1] for i in range(len(cs) - 1) if cs[i + 1][2] == "force"]
        gb = [cs[i + 1][0] - cs[i][1] for i in range(len(cs) - 1) if cs[i + 1][2] == "bin"]
        end = max(b for _, _, b in rows)
        print(f"  {f.split('.')[-2]}: start {cs[0][0]:7.2f} end {end:8.2f} busy {busy:7.2f} (force {force:7.2f}) "
              f"gaps {sum(gaps):6.2f} [before force {sum(gf):6.2f} n={len(gf)}, before bin {sum(gb):5.2f}] "
              f"largest {['%.2f' % g for g in big]} hop {hop:6.2f}")
