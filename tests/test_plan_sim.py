"""CPU simulation of the ring's stage plans (dsea_plan_ops, the op lists run_plan
executes) across all ranks, with the cross-rank data dependencies of the peer
ring: a worker-0 force/pass of rank r waits until the predecessor's last worker has
delivered (binned or passed through) every slot it reads for that super-cycle;
everything else is ordered by the rank's own stream.  Checks, for many (N_S, N_GPU,
W, B): no deadlock -- in particular beyond Eq. (1)'s N_max, where the ring must run
at the plateau (Q17) rather than stall -- local inputs binned before use,
and every (slice, timestep) unit computed exactly once (Q15)."""
import itertools

import pytest

from paper_2507_11289_b200 import dsea as D

R, F, P, BN, S = D.OP_RECV, D.OP_FORCE, D.OP_PASS, D.OP_BIN, D.OP_SEND


def simulate(ns, ng, W, n_steps, B):
    plans = [D.dsea_plan_ops(ns, ng, r, W, n_steps, B) for r in range(ng)]
    ptr = [0] * ng
    # deliveries[r][s]: times slot s of rank r's input buffer was filled by the predecessor
    deliveries = [[0] * ns for _ in range(ng)]
    # binned[r][w][s]: times worker w of rank r finalised slot s (its output buffer)
    binned = [[[0] * ns for _ in range(W)] for _ in range(ng)]
    done_units = {}
    progress = True
    while progress:
        progress = False
        for r in range(ng):
            while ptr[r] < len(plans[r]):
                kind, stage, w, j, n, K, t = (int(v) for v in plans[r][ptr[r]])
                if kind in (F, P):
                    lo = max(j - 1, 0)
                    hi = min(j + n, ns - 1) if kind == F else j + n - 1
                    if w == 0:
                        if ng > 1 and not (r == 0 and K == 0):
                            need = K + 1 if r > 0 else K
                            if any(deliveries[r][s] < need for s in range(lo, hi + 1)):
                                break          # blocked on the ring
                    else:
                        # local input: worker w-1's output of this super-cycle, already
                        # binned earlier in this rank's stream
                        assert all(binned[r][w - 1][s] >= K + 1 for s in range(lo, hi + 1)), \
                            ("local order", r, stage, w, j, K)
                    if kind == F:
                        for s in range(j, j + n):
                            key = (s, t)
                            assert key not in done_units, ("unit twice", key, r)
                            done_units[key] = r
                    else:
                        for s in range(j, j + n):
                            binned[r][w][s] += 1
                            if w == W - 1 and ng > 1:
                                deliveries[(r + 1) % ng][s] += 1
                elif kind == BN:
                    for s in range(j, j + n):
                        binned[r][w][s] += 1
                        if w == W - 1 and ng > 1:
                            deliveries[(r + 1) % ng][s] += 1
                ptr[r] += 1
                progress = True
    stuck = [r for r in range(ng) if ptr[r] < len(plans[r])]
    return stuck, done_units, deliveries


CASES = [(ns, ng, W, B) for ns, ng, W, B in itertools.product(
    (6, 8, 12, 13, 16, 24, 32, 48, 64), (2, 3, 4, 8), (1, 2, 3), (1, 2, 3, 4, 8))
    if B <= ns and ns >= 2 + 2 * W]


@pytest.mark.parametrize("ns,ng,W,B", CASES)
def test_ring_plan_completes_and_covers_every_unit(ns, ng, W, B):
    cycles = 3
    n_steps = cycles * ng * W - (W > 1)      # not a multiple of N_w: pass-through (Q15)
    stuck, units, deliveries = simulate(ns, ng, W, n_steps, B)
    assert not stuck, f"deadlock: ranks {stuck} blocked (ns={ns} ng={ng} W={W} B={B})"
    assert len(units) == ns * n_steps
    assert set(units) == {(s, t) for s in range(ns) for t in range(n_steps)}
    # the state returns to rank 0 after the last super-cycle (Q22)
    assert all(d == cycles for d in deliveries[0])


# the benchmark's ring configurations (C4: 109 slices, auto B = 7 at 2/4 GPUs, 4 at 8;
# C3: 256 slices) including the lead blocks of make_blocks
BENCH_CASES = [(109, 2, 1, 7), (109, 4, 1, 7), (109, 8, 1, 4), (109, 4, 2, 5), (256, 8, 1, 7), (20, 2, 1, 6)]


@pytest.mark.parametrize("lead", ["0", "1"])
@pytest.mark.parametrize("ns,ng,W,B", BENCH_CASES)
def test_bench_ring_plans(ns, ng, W, B, lead, monkeypatch):
    monkeypatch.setenv("DSEA_LEAD_BLOCKS", lead)
    n_steps = 2 * ng * W
    stuck, units, deliveries = simulate(ns, ng, W, n_steps, B)
    assert not stuck
    assert set(units) == {(s, t) for s in range(ns) for t in range(n_steps)}
    assert all(d == 2 for d in deliveries[0])


@pytest.mark.parametrize("ns,ng,B,lead", [(109, 4, 7, True), (109, 8, 4, True), (109, 1, 7, False),
                                          (109, 4, 3, False), (11, 2, 4, False), (20, 2, 6, True)])
def test_lead_blocks(ns, ng, B, lead, monkeypatch):
    """Blocks are balanced (ceil(N_S / B) blocks whose sizes differ by at most one, so
    no short tail block); with DSEA_LEAD_BLOCKS=1 on a ring the first two blocks of a
    super-cycle hold 2 slices (shorter per-rank pipeline lag), the rest balanced."""
    monkeypatch.setenv("DSEA_LEAD_BLOCKS", "1")
    ops = D.dsea_plan_ops(ns, ng, 0, 1, ng, B)
    sizes = [int(o[4]) for o in ops if int(o[0]) in (F, P) and int(o[5]) == 0]
    assert sum(sizes) == ns
    rest = sizes[2:] if lead else sizes
    if lead:
        assert sizes[:2] == [2, 2]
    assert len(rest) == -(-(ns - (4 if lead else 0)) // B)
    assert max(rest) <= B and max(rest) - min(rest) <= 1
    assert all(sz >= 2 for sz in sizes)


def _pushes(ops, W):
    """(cycle, slot) of every slot the last worker pushes to the ring successor, in op order."""
    out = []
    for kind, stage, w, j, n, K, t in (tuple(int(v) for v in o) for o in ops):
        if w == W - 1 and kind in (BN, P):
            out += [(K, s) for s in range(j, j + n)]
    return out


@pytest.mark.parametrize("ns,ng,W,B", CASES[::7] + BENCH_CASES)
def test_pushes_leave_in_slot_order(ns, ng, W, B):
    """What the monotone ring counters rely on (order_pushes): each rank
    pushes every slot once per super-cycle, in strictly increasing (super-cycle, slot)
    order -- including partial super-cycles passed through (Q15) -- and the successor's
    receives come in the same slot order."""
    for n_steps in (2 * ng * W, 2 * ng * W - 1, 3 * ng * W - (W > 1)):
        plans = [D.dsea_plan_ops(ns, ng, r, W, n_steps, B) for r in range(ng)]
        for r in range(ng):
            p = _pushes(plans[r], W)
            assert p == sorted(p) and len(set(p)) == len(p), (r, n_steps)
            cycles = -(-n_steps // (ng * W))
            assert len(p) == cycles * ns
            recv = [int(o[3]) for o in plans[(r + 1) % ng] if int(o[0]) == R]
            assert recv == [s for _, s in p]      # (rank 0 also takes the last cycle back, Q22)


def _staging_pool_hazards(ops, ns, pool, seq=True):
    """Walk one rank's ops in stream order (force passes and bins run on the compute
    stream in plan order): a FORCE (worker w, cycle K, slices [j, j+n)) writes staging
    entries (K, j..j+n-1) of worker w into slots (K N_S + s) mod pool; a BIN of cycle K
    over [m, m+n) reads (K, max(m-1, 0) .. min(m+n, N_S-1)) (atoms move at most one
    slice per step).  Returns the writes that land on a slot whose current occupant
    still has a read ahead of it."""
    ops = [tuple(int(v) for v in o) for o in ops]
    last_read = {}                               # (w, K, s) -> index of the last BIN reading it
    for i, (kind, _, w, j, n, K, _) in enumerate(ops):
        if kind == BN:
            for s in range(max(j - 1, 0), min(j + n, ns - 1) + 1):
                last_read[(w, K, s)] = i
    occupant = {}                                # (w, slot) -> (K, s)
    bad = []
    for i, (kind, _, w, j, n, K, _) in enumerate(ops):
        if kind != F:
            continue
        for s in range(j, j + n):
            slot = (K * ns + s) % pool if seq else s % pool
            prev = occupant.get((w, slot))
            if prev is not None and prev != (K, s) and last_read.get((w, *prev), -1) > i:
                bad.append((i, (K, s), prev))
            occupant[(w, slot)] = (K, s)
    return bad


@pytest.mark.parametrize("ns,ng,W,B", CASES[::3] + BENCH_CASES)
def test_staging_pool_size_never_overwrites_a_live_slice(ns, ng, W, B):
    """NEXT-3 slot pools: a staged-schedule worker's staging buffer holds
    2 B_max + 4 slices in slots that follow the global sequence number K N_S + j, with no
    runtime guard -- only the compute stream's order.  For every plan (rings of 1-8
    ranks, W workers, B slices per stage, partial super-cycles), no force pass may
    overwrite a staging slot whose occupant a later bin still reads.  The same plans
    with slot = j mod pool (no sequence number) do overwrite: the previous super-cycle's
    last slice is binned after the next cycle's first block."""
    for n_steps in (ng * W * 2 + 1, ng * W * 3):
        for r in range(ng):
            ops = D.dsea_plan_ops(ns, ng, r, W, n_steps, B)
            bmax = max(int(o[4]) for o in ops if int(o[0]) == F)
            pool = min(ns, 2 * bmax + 4)
            assert not _staging_pool_hazards(ops, ns, pool), (ns, ng, W, B, r, n_steps)


def test_staging_pool_needs_the_sequence_number():
    """The negative control of the test above: with slot = j mod pool the last slice of
    one super-cycle and the first block of the next collide (found on B200 as a failing
    staged ring of one: P8, W = 1, B = 3)."""
    ns, ng, W, B = 32, 1, 1, 3
    ops = D.dsea_plan_ops(ns, ng, 0, W, 7, B)
    pool = 2 * B + 4
    assert _staging_pool_hazards(ops, ns, pool, seq=False)
    assert not _staging_pool_hazards(ops, ns, pool, seq=True)


def _nccl_sim():
    import importlib.util
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts", "nccl_plan_sim.py")
    spec = importlib.util.spec_from_file_location("nccl_plan_sim", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _degenerate(ns, B):
    return -(-ns // B) <= 2          # one or two blocks per super-cycle


@pytest.mark.parametrize("ns,ng,W,B", [c for c in CASES[::5] if c[1] > 1 and not _degenerate(c[0], c[3])]
                         + [(32, 4, 2, 3), (32, 4, 1, 5)])
def test_nccl_plans_have_no_stream_level_deadlock(ns, ng, W, B):
    """The NCCL comparison backend's streams (compute, send, receive) with event waits
    bound at enqueue time and rendezvous p2p groups matched in posting order
    (`scripts/nccl_plan_sim.py`): every plan with more than two blocks per super-cycle
    completes -- including the two 4-GPU plateau cases that hang on B200, whose hang is
    therefore not a stream-level cycle of the plan (the ranks that never return block on
    the host inside NCCL).  With one or two blocks per super-cycle at the
    plateau the model does deadlock (grouped rendezvous sends; the peer backend, which
    needs no rendezvous, completes them): a limitation of the comparison backend only --
    the automatic block size always gives >= N_GPU (2 + W) - 1 blocks."""
    sim = _nccl_sim()
    for n_steps in (ng * W, ng * W * 2 + 1):
        assert not sim.simulate(ns, ng, W, n_steps, B), (ns, ng, W, B, n_steps)


def test_nccl_model_finds_the_degenerate_plateau_deadlock():
    """Negative control of the NCCL stream model: 16 slices in blocks of 8 on a ring of 3
    (two blocks per super-cycle, a partial last cycle) deadlocks under rendezvous
    semantics -- so the model can find a cycle when there is one."""
    assert _nccl_sim().simulate(16, 3, 1, 7, 8)
