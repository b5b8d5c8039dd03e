"""Stream-level simulation of the NCCL comparison backend of run_plan (dsea_host.cpp):
every rank's compute / send / receive streams as FIFO queues of kernels, event records,
event waits (bound, like cudaStreamWaitEvent, to the latest record enqueued before the
wait) and grouped NCCL p2p operations with rendezvous semantics (a message completes
when both its send and its receive group have been posted on their streams; a group
completes when all its messages have).  Messages on a link are matched in posting order.

Reports whether the op lists dsea_plan_ops returns can deadlock at the GPU level under
these semantics (a host-side block inside NCCL is not modelled).

  python scripts/nccl_plan_sim.py                 # the known cases
  python scripts/nccl_plan_sim.py 32 4 2 3 12     # ns ng W B steps"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11289_b200 import dsea as D  # noqa: E402

R, F, P, BN, S = D.OP_RECV, D.OP_FORCE, D.OP_PASS, D.OP_BIN, D.OP_SEND


def build_queues(ns, ng, W, n_steps, B):
    """Per rank, the items run_plan enqueues on its compute (cs), send (ss) and
    receive (rs) streams, in host order."""
    ranks = []
    for r in range(ng):
        ops = [tuple(int(v) for v in o) for o in D.dsea_plan_ops(ns, ng, r, W, n_steps, B)]
        q = {"cs": [], "ss": [], "rs": []}
        rec = defaultdict(int)                     # event name -> records enqueued so far
        sent = set()

        def record(stream, ev):
            rec[ev] += 1
            q[stream].append(("record", ev, rec[ev]))

        def wait(stream, ev):
            if rec[ev]:
                q[stream].append(("wait", ev, rec[ev]))

        i = 0
        while i < len(ops):
            kind, stage, w, j, n, K, t = ops[i]
            if kind == R:
                e = i
                while e < len(ops) and ops[e][0] == R and ops[e][1] == stage:
                    e += 1
                sl = [ops[k][3] for k in range(i, e)]
                for s in sl:
                    wait("rs", ("free", s))
                q["rs"].append(("nccl", "recv", tuple(sl)))
                for s in sl:
                    record("rs", ("recv", s))
                i = e
                continue
            if kind == S:
                e = i
                while e < len(ops) and ops[e][0] == S and ops[e][1] == stage:
                    e += 1
                sl = [ops[k][3] for k in range(i, e)]
                for s in sl:
                    wait("ss", ("bin", s))
                q["ss"].append(("nccl", "send", tuple(sl)))
                for s in sl:
                    record("ss", ("send", s))
                    sent.add(s)
                i = e
                continue
            if kind == F:
                if w == 0 and ng > 1 and not (r == 0 and K == 0):
                    wait("cs", ("recv", min(j + n, ns - 1)))
                q["cs"].append(("kernel", "force", (w, j, n, K)))
                if w == 0 and ng > 1:
                    f0, f1 = max(j - 1, 0), (ns - 1 if j + n == ns else j + n - 2)
                    for s in range(f0, f1 + 1):
                        record("cs", ("free", s))
            elif kind == P:
                if w == 0 and ng > 1 and not (r == 0 and K == 0):
                    wait("cs", ("recv", j + n - 1))
                if w == W - 1 and ng > 1:
                    for s in range(j, j + n):
                        if s in sent:
                            wait("cs", ("send", s))
                q["cs"].append(("kernel", "pass", (w, j, n, K)))
                if w == 0 and ng > 1:
                    for s in range(j, j + n):
                        record("cs", ("free", s))
                if w == W - 1 and ng > 1:
                    for s in range(j, j + n):
                        record("cs", ("bin", s))
            elif kind == BN:
                if w == W - 1 and ng > 1:
                    for s in range(j, j + n):
                        if s in sent:
                            wait("cs", ("send", s))
                q["cs"].append(("kernel", "bin", (w, j, n, K)))
                if w == W - 1 and ng > 1:
                    for s in range(j, j + n):
                        record("cs", ("bin", s))
            i += 1
        ranks.append(q)
    return ranks


def simulate(ns, ng, W, n_steps, B):
    ranks = build_queues(ns, ng, W, n_steps, B)
    done_rec = [defaultdict(int) for _ in range(ng)]    # event -> highest record completed
    ptr = [{k: 0 for k in ("cs", "ss", "rs")} for _ in range(ng)]
    # message matching: link g carries rank g -> g+1; k-th send message == k-th recv message
    posted = defaultdict(lambda: [0, 0])                 # (link, msg) -> [send posted, recv posted]
    next_msg = defaultdict(lambda: [0, 0])               # link -> [next send idx, next recv idx]
    group_msgs = {}                                      # (rank, stream, ptr) -> list of (link, msg)
    progress = True
    while progress:
        progress = False
        for r in range(ng):
            for st in ("cs", "ss", "rs"):
                q = ranks[r][st]
                while ptr[r][st] < len(q):
                    it = q[ptr[r][st]]
                    if it[0] == "kernel":
                        pass
                    elif it[0] == "record":
                        done_rec[r][it[1]] = max(done_rec[r][it[1]], it[2])
                    elif it[0] == "wait":
                        if done_rec[r][it[1]] < it[2]:
                            break
                    else:                               # nccl group: post, then wait for all
                        key = (r, st, ptr[r][st])
                        if key not in group_msgs:
                            side = 0 if it[1] == "send" else 1
                            link = r if side == 0 else (r - 1) % ng
                            msgs = []
                            for _ in it[2]:
                                m = next_msg[link][side]
                                next_msg[link][side] += 1
                                posted[(link, m)][side] = 1
                                msgs.append((link, m))
                            group_msgs[key] = msgs
                            progress = True
                        if not all(posted[lm][0] and posted[lm][1] for lm in group_msgs[key]):
                            break
                    ptr[r][st] += 1
                    progress = True
    stuck = {(r, st): ranks[r][st][ptr[r][st]] for r in range(ng) for st in ("cs", "ss", "rs")
             if ptr[r][st] < len(ranks[r][st])}
    return stuck


if __name__ == "__main__":
    if len(sys.argv) > 1:
        cases = [tuple(int(a) for a in sys.argv[1:6])]
    else:
        # (ns, ng, W, B, steps): the two hanging 4-GPU cases, then passing controls
        cases = [(32, 4, 2, 3, 12), (32, 4, 1, 5, 12), (32, 2, 1, 1, 16), (32, 2, 2, 3, 10), (32, 4, 1, 2, 16),
                 (32, 4, 2, 3, 4)]
    for ns, ng, W, B, steps in cases:
        stuck = simulate(ns, ng, W, steps, B)
        print(f"ns={ns} ng={ng} W={W} B={B} steps={steps}: "
              + ("completes" if not stuck else f"DEADLOCK, heads: {dict(list(stuck.items())[:6])}"))
