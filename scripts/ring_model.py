"""Timing model of the MD ring: a discrete-event simulation of every rank's compute
stream over the real stage plan (dsea_plan_ops), calibrated on the measured B200 runs.

  python scripts/ring_model.py [n_gpus ...]

Per rank, ops run in plan order on one compute stream.  A worker-0 FORCE/PASS waits
until the slots it reads have arrived; the last worker's BIN (or PASS) pushes slices
to the successor, which arrive after the copy (bytes / NVLink bandwidth) plus a fixed
latency, in push order.  Durations (C4, measured on one B200 unless noted):
  force  = per-slice fused time x slices + per-launch overhead
  bin    = per-slice fused time x slices + per-launch overhead
  push   = slice bytes / copy bandwidth + latency (hop stream, overlaps compute)
Releases are not modelled (every rank has a slot per slice, so pushes never wait)."""
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2507_11289_b200 import dsea as D  # noqa: E402

NS = 109
# round-2 final kernels (profiles/r02/bench_c4_n1.json, launches_bench_n1.csv); round 1:
# force 9.85 ms, bins 0.88 ms
T_FORCE_SLICE = 8.40 / NS          # ms, fused C4 force launch / 109 slices
T_BIN_SLICE = 0.79 / NS            # ms, fused C4 bins / 109 slices
T_FORCE_LAUNCH = 0.022             # ms per force launch (ramp + tail; timeline)
T_BIN_LAUNCH = 0.025               # ms per bin run (3 kernels + gaps)
SLICE_BYTES = 11.4e6
COPY_BW = 4.0e8                    # bytes/ms (~400 GB/s per copy-engine hop, timeline)
HOP_LAT = 0.010                    # ms (flags, stream waits)


def auto_block(ng, W=1, n_atoms=16_384_000):
    import math
    nb_t = math.ceil(n_atoms / 2.0e6)
    depth = ng * (2 + W) - 1 if ng > 1 else 2 + W
    nb = max(nb_t, depth)
    B = max(1, -(-NS // nb))
    while B > 1 and -(-NS // B) < depth:
        B -= 1
    return B


def simulate(ng, cycles=10, W=1, B=None):
    B = B or auto_block(ng, W)
    n_steps = cycles * ng * W
    plans = [[tuple(int(v) for v in o) for o in D.dsea_plan_ops(NS, ng, r, W, n_steps, B)] for r in range(ng)]
    arrivals = [[[] for _ in range(NS)] for _ in range(ng)]   # per rank, per slot: arrival times in order
    used = [[0] * NS for _ in range(ng)]
    clock = [0.0] * ng
    hop_free = [0.0] * ng
    ptr = [0] * ng
    busy = [0.0] * ng
    progress = True
    while progress:
        progress = False
        for r in range(ng):
            while ptr[r] < len(plans[r]):
                kind, stage, w, j, n, K, t = plans[r][ptr[r]]
                start = clock[r]
                if kind in (1, 2) and w == 0 and not (r == 0 and K == 0):
                    need = min(j + n, NS - 1) if kind == 1 else j + n - 1
                    lo = max(j - 1, 0)
                    k_needed = K if r == 0 else K + 1
                    # arrivals counted per slot: the (k_needed)-th arrival of every slot read
                    ok = all(len(arrivals[r][s]) >= k_needed for s in range(lo, need + 1))
                    if not ok:
                        break
                    start = max(start, max(arrivals[r][s][k_needed - 1] for s in range(lo, need + 1)))
                if kind == 1:
                    dur = T_FORCE_SLICE * n + T_FORCE_LAUNCH
                elif kind == 3:
                    dur = T_BIN_SLICE * n + T_BIN_LAUNCH
                elif kind == 2:
                    dur = 0.002 * n
                else:
                    dur = 0.0
                end = start + dur
                busy[r] += dur
                clock[r] = end
                if ng > 1 and w == W - 1 and kind in (2, 3):
                    s_ = hop_free[r] = max(hop_free[r], end) + SLICE_BYTES * n / COPY_BW + HOP_LAT
                    for s in range(j, j + n):
                        arrivals[(r + 1) % ng][s].append(s_)
                ptr[r] += 1
                progress = True
    assert all(ptr[r] == len(plans[r]) for r in range(ng)), "deadlock in model"
    makespan = max(clock)
    if ng > 1:
        makespan = max(makespan, max(a[-1] for a in arrivals[0] if a))   # state back on rank 0
    atom_steps = 16_384_000 * n_steps
    return atom_steps / (makespan * 1e-3), makespan, B


if __name__ == "__main__":
    one = 16_384_000 / ((T_FORCE_SLICE + T_BIN_SLICE) * NS * 1e-3)
    print(f"model 1 GPU (fused): {one:.3e} atom-timesteps/s (measured 1.776e9; ring4_final: 2 GPUs 90.5 %, "
          f"4 GPUs 84.9 % of N x one GPU)")
    for ng in [int(a) for a in sys.argv[1:]] or [2, 4, 8]:
        v, ms, B = simulate(ng)
        print(f"model {ng} GPUs, B = {B}: {v:.3e} atom-timesteps/s = {v / (ng * one):.1%} of {ng} x 1 GPU "
              f"({ms:.1f} ms for 10 super-cycles)")
