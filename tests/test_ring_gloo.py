"""World-size-2 `gloo` tests of the N>1 ring path on CPU (no GPU needed).

1. The schedule each rank derives on its own (dsea_schedule) matches across ranks:
   what rank g sends is what rank g+1 receives, in order (§3.1).
2. Ring bootstrap plumbing: rank 0's NCCL link ids reach every rank unchanged.
3. A CPU emulation of the ring data flow: two gloo ranks execute their stage
   schedules literally -- receive, process slice j from slices j-1, j, j+1 of the
   same timestep (O_in = 1), finalise slice j-1 from the contributions of j-2..j
   (O_out = 1), pass finished slices to the successor -- with the oracle's pair law
   as the worker kernel.  After 2 super-cycles (4 timesteps) the state equals the
   whole-domain oracle run: the ring is an exact re-scheduling of timesteps (P:55,
   P:86), which is what the GPU ring relies on.
"""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2507_11289_b200 import dsea as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(fn, world, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_entry, args=(fn, r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, res = q.get(timeout=300)
        out[r] = res
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        if isinstance(out[r], BaseException) or (isinstance(out[r], str) and out[r].startswith("ERR")):
            raise AssertionError(f"rank {r}: {out[r]}")
    return out


def _entry(fn, rank, world, port, q, *args):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        res = fn(rank, world, *args)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, res))
    except BaseException as e:  # report, don't hang the parent
        import traceback
        q.put((rank, "ERR " + traceback.format_exc()))


# ---------------------------------------------------------------- 1. schedules
def _schedule_worker(rank, world, ns, W, cycles):
    rows = D.dsea_schedule(ns, world, rank, W, cycles)
    sends = [int(r[5]) for r in rows if r[5] > 0 and r[2] == W - 1]
    recvs = [int(r[1]) for r in rows if r[1] > 0]
    units = [(int(r[3]), int(r[7])) for r in rows if r[2] >= 0 and r[3] > 0]
    allv = [None] * world
    dist.all_gather_object(allv, (sends, recvs, units))
    for g in range(world):
        nxt = (g + 1) % world
        got = allv[nxt][1][ns:] if nxt == 0 else allv[nxt][1]
        if allv[g][0] != got:
            return f"ERR send/recv mismatch {g}->{nxt}"
    all_units = sorted(u for a in allv for u in a[2])
    want = sorted((j, t) for j in range(1, ns + 1) for t in range(cycles * world * W))
    return "ok" if all_units == want else "ERR units"


@pytest.mark.parametrize("W", [1, 2])
def test_gloo_schedules_match(W):
    res = _spawn(_schedule_worker, 2, 12, W, 3)
    assert all(v == "ok" for v in res.values())


# ---------------------------------------------------------------- 2. bootstrap
def _bootstrap_worker(rank, world):
    try:
        ids = [b"".join(D.dsea_ring_unique_id() for _ in range(world))] if rank == 0 else [None]
    except D.DseaError:
        ids = [b"x" * (D.NCCL_ID_BYTES * world)] if rank == 0 else [None]  # NCCL not loadable here
    dist.broadcast_object_list(ids, src=0)
    digest = [None] * world
    dist.all_gather_object(digest, (len(ids[0]), hashlib.sha256(ids[0]).hexdigest()))
    return "ok" if len(set(digest)) == 1 and digest[0][0] == D.NCCL_ID_BYTES * world else "ERR"


def test_gloo_ring_id_broadcast():
    res = _spawn(_bootstrap_worker, 2)
    assert all(v == "ok" for v in res.values())


# ---------------------------------------------------------------- 3. ring emulation
NX, NY, NZ, NS, RC, DT = 16, 5, 5, 8, 2.5, 0.0018


def _geometry():
    return oracle.geometry(NX, NY, NZ, 0.8, RC, NS, 1)


def _initial():
    g = _geometry()
    x = oracle.lattice(NX, NY, NZ, g.a)
    v = oracle.velocities(len(x), 17, 1.0)
    return g, x, v


def _slice_of(x, g):
    _, sl = oracle.bin_atoms(x, g.l, g.cells, 1)
    return sl


def _pack(rows):
    """slice record: (n, 10) = id, x, y, z, vx, vy, vz, fx, fy, fz"""
    return np.ascontiguousarray(rows, dtype=np.float64)


def _unit(g, left, mid, right):
    """Worker kernel for one slice: Algorithm 1 force on the atoms of `mid` from
    the atoms of left+mid+right (oracle pair law), kick, drift, walls; returns the
    advanced atoms of `mid` with their destination slice."""
    parts = [p for p in (left, mid, right) if p is not None]
    allr = np.concatenate(parts)
    F, _, _ = oracle.forces(allr[:, 1:4], g.b, RC, nthreads=1)
    off = 0 if left is None else len(left)
    m = mid.copy()
    Fn = F[off:off + len(mid)]
    m[:, 4:7] = m[:, 4:7] + (Fn + m[:, 7:10]) * 0.5 * DT
    m[:, 1:4] = m[:, 1:4] + m[:, 4:7] * DT + Fn * 0.5 * (DT * DT)
    m[:, 7:10] = Fn
    lo = m[:, 1] < 0
    hi = m[:, 1] > g.b[0]
    m[lo, 1] = -m[lo, 1]
    m[hi, 1] = 2 * g.b[0] - m[hi, 1]
    m[lo | hi, 4] *= -1
    m[lo | hi, 7] *= -1
    for d in (2, 3):
        b = g.b[d - 1]
        m[m[:, d] < 0, d] += b
        m[m[:, d] >= b, d] -= b
    return m, _slice_of(m[:, 1:4], g)


def _ring_worker(rank, world, cycles):
    g, x, v = _initial()
    ns = NS
    rows = D.dsea_schedule(ns, world, rank, 1, cycles)
    nxt, prv = (rank + 1) % world, (rank - 1) % world
    inbuf = {}
    if rank == 0:
        sl = _slice_of(x, g)
        ids = np.arange(len(x))
        for j in range(ns):
            sel = sl == j
            inbuf[j] = _pack(np.column_stack([ids[sel], x[sel], v[sel], np.zeros((sel.sum(), 3))]))
    staged = {}   # item -> (atoms, dest)
    out = {}
    pending = []
    for st, recv, w, proc, binned, send, cyc, t in rows:
        if recv > 0 and not (rank == 0 and cyc == 0):
            n = np.zeros(1, dtype=np.int64)
            dist.recv(_t(n), src=prv)
            buf = np.zeros((int(n[0]), 10))
            if n[0]:
                dist.recv(_t(buf), src=prv)
            inbuf[recv - 1] = buf
        if w >= 0 and proc > 0:
            j = proc - 1
            staged[j] = _unit(g, inbuf.get(j - 1) if j > 0 else None, inbuf[j],
                              inbuf.get(j + 1) if j < ns - 1 else None)
        if w >= 0 and binned > 0:
            m = binned - 1
            parts = [staged[s][0][staged[s][1] == m] for s in (m - 1, m, m + 1) if s in staged]
            rec = np.concatenate(parts)
            out[m] = rec[np.argsort(rec[:, 0], kind="stable")]
        if w >= 0 and send > 0:
            m = send - 1
            rec = out[m]
            pending.append(dist.isend(_t(np.array([len(rec)], dtype=np.int64)), dst=nxt))
            if len(rec):
                pending.append(dist.isend(_t(rec), dst=nxt))
    for p in pending:
        p.wait()
    if rank == 0:
        final = np.concatenate([inbuf[j] for j in range(ns)])
        return final[np.argsort(final[:, 0])]
    return "ok"


def _t(a):
    import torch
    return torch.from_numpy(a)


def test_gloo_ring_emulation_equals_sequential():
    world, cycles = 2, 2
    res = _spawn(_ring_worker, world, cycles)
    final = res[0]
    g, x, v = _initial()
    xo, vo, Fo, _ = oracle.run(x, v, np.zeros_like(x), g.b, RC, DT, world * cycles)
    assert final.shape == (len(x), 10)
    assert np.array_equal(final[:, 0], np.arange(len(x)))
    d = final[:, 1:4] - xo
    d[:, 1:] -= g.b[1:] * np.round(d[:, 1:] / g.b[1:])
    assert np.max(np.abs(d)) < 1e-12
    assert np.max(np.abs(final[:, 4:7] - vo)) < 1e-11


# ---------------------------------------------------------------- 4. stencil ring emulation
# The second workload (include/dsea_grid.h: O_in = 1, O_out = 0) on two
# gloo ranks, executing the shared stage plan (dsea_plan_ops) op by op the way
# dsea_grid.cpp does: FORCE = the oracle FTCS step of a block's planes from the
# worker's input buffer into its output buffer; BIN = the last worker pushes the
# finished slices to the successor (one message per slice); PASS = copy through /
# push (partial super-cycles, Q15).  Pushes leave in (super-cycle, slot) order: a BIN
# of the previous cycle listed after a PASS of the same stage goes first (the rule
# dsea_grid.cpp applies for its monotone counters).  Receives are consumed lazily, in
# order, when a worker-0 op needs a slot.  The field on rank 0 must equal the
# sequential oracle run bit for bit.
GNX, GNY, GNZ, GNS, GR = 24, 4, 5, 12, 0.12
R_, F_, P_, BN_, S_ = D.OP_RECV, D.OP_FORCE, D.OP_PASS, D.OP_BIN, D.OP_SEND


def _grid_ring_worker(rank, world, W, B, n_steps, calls):
    from oracle import grid as OG
    from tests import inputs
    p = GNX // GNS
    u0 = inputs.grid_field(GNX, GNY, GNZ, 3)
    inb = u0.copy() if rank == 0 else np.zeros_like(u0)
    outb = [np.zeros_like(u0) for _ in range(W)]
    nxt, prv = (rank + 1) % world, (rank - 1) % world
    pending, queue = [], []          # isend handles; expected receives (slot) in order
    got = {}                          # slot -> times received

    expected = {}                     # slot -> receptions the plan has announced so far

    def recv_until(slot):
        while got.get(slot, 0) < expected.get(slot, 0):
            s = queue.pop(0)
            buf = np.zeros((p, GNY, GNZ))
            dist.recv(_t(buf), src=prv)
            inb[s * p:(s + 1) * p] = buf
            got[s] = got.get(s, 0) + 1

    def push(src, m, n):
        for s in range(m, m + n):
            pending.append(dist.isend(_t(np.ascontiguousarray(src[s * p:(s + 1) * p])), dst=nxt))

    per = n_steps // calls
    for call in range(calls):
        steps = per if call < calls - 1 else n_steps - per * (calls - 1)
        ops = [tuple(int(v) for v in o) for o in D.dsea_plan_ops(GNS, world, rank, W, steps, B)]
        for i in range(len(ops) - 1):   # push order rule (see above)
            if ops[i][0] == P_ and ops[i][2] == W - 1:
                k = i + 1
                while k < len(ops) and ops[k][1] == ops[i][1] and ops[k][2] == ops[i][2] and ops[k][0] == BN_:
                    if ops[k][5] < ops[i][5]:
                        ops.insert(i, ops.pop(k))
                        i += 1
                    k += 1
        for kind, stage, w, j, n, K, t in ops:
            if kind == R_:
                queue.append(j)
                expected[j] = expected.get(j, 0) + 1
            elif kind in (F_, P_):
                src = inb if w == 0 else outb[w - 1]
                if w == 0:
                    recv_until(min(j + n, GNS - 1) if kind == F_ else j + n - 1)
                if kind == F_:
                    lo, hi = max(j * p - 1, 0), min((j + n) * p + 1, GNX)
                    res = OG.ftcs_step(src[lo:hi], GR)
                    outb[w][j * p:(j + n) * p] = res[j * p - lo:j * p - lo + n * p]
                elif w == W - 1:
                    push(src, j, n)
                else:
                    outb[w][j * p:(j + n) * p] = src[j * p:(j + n) * p]
            elif kind == BN_ and w == W - 1:
                push(outb[W - 1], j, n)
        if rank == 0:                 # the final super-cycle lands on rank 0
            recv_until(GNS - 1)
    for h in pending:
        h.wait()
    return inb if rank == 0 else "ok"


@pytest.mark.parametrize("W,B,n_steps,calls", [(1, 2, 6, 1), (1, 3, 7, 2), (2, 1, 8, 1), (2, 4, 9, 2), (1, 1, 5, 1)])
def test_gloo_stencil_ring_emulation_equals_sequential(W, B, n_steps, calls):
    from oracle import grid as OG
    from tests import inputs
    res = _spawn(_grid_ring_worker, 2, W, B, n_steps, calls)
    u0 = inputs.grid_field(GNX, GNY, GNZ, 3)
    assert np.array_equal(res[0], OG.run(u0, GR, n_steps))


# ---------------------------------------------------------------- 5. MD ring emulation, general plan
# The MD workload (O_in = O_out = 1) on two gloo ranks executing dsea_plan_ops -- blocks
# of B slices, W workers per rank, split calls and partial super-cycles -- op by op:
# FORCE advances each slice of the block from its neighbours (oracle pair law, _unit);
# BIN finalises a slice from the staged contributions of slices s-1..s+1; PASS copies
# a block through; the last worker pushes finalised slices to the successor (one
# message per slice, in the order dsea_plan_ops returns).  Equals the whole-domain
# oracle run.
def _md_plan_worker(rank, world, W, B, n_steps, calls):
    g, x, v = _initial()
    ns = NS
    nxt, prv = (rank + 1) % world, (rank - 1) % world
    inb = {}
    if rank == 0:
        sl = _slice_of(x, g)
        ids = np.arange(len(x))
        for j in range(ns):
            sel = sl == j
            inb[j] = _pack(np.column_stack([ids[sel], x[sel], v[sel], np.zeros((sel.sum(), 3))]))
    out = [dict() for _ in range(W)]
    staged = [dict() for _ in range(W)]
    pending, queue, got, expected = [], [], {}, {}

    def recv_until(slot):
        while got.get(slot, 0) < expected.get(slot, 0):
            s = queue.pop(0)
            n = np.zeros(1, dtype=np.int64)
            dist.recv(_t(n), src=prv)
            buf = np.zeros((int(n[0]), 10))
            if n[0]:
                dist.recv(_t(buf), src=prv)
            inb[s] = buf
            got[s] = got.get(s, 0) + 1

    def push(rec):
        pending.append(dist.isend(_t(np.array([len(rec)], dtype=np.int64)), dst=nxt))
        if len(rec):
            pending.append(dist.isend(_t(np.ascontiguousarray(rec)), dst=nxt))

    per = n_steps // calls
    for call in range(calls):
        steps = per if call < calls - 1 else n_steps - per * (calls - 1)
        for kind, stage, w, j, n, K, t in (tuple(int(q) for q in o) for o in D.dsea_plan_ops(ns, world, rank, W, steps, B)):
            if kind == R_:
                queue.append(j)
                expected[j] = expected.get(j, 0) + 1
                continue
            src = inb if w == 0 else out[w - 1]
            if kind in (F_, P_) and w == 0:
                recv_until(min(j + n, ns - 1) if kind == F_ else j + n - 1)
            if kind == F_:
                for s in range(j, j + n):
                    staged[w][s] = _unit(g, src.get(s - 1) if s > 0 else None, src[s],
                                         src.get(s + 1) if s < ns - 1 else None)
            elif kind == P_:
                for s in range(j, j + n):
                    out[w][s] = src[s]
                    if w == W - 1:
                        push(src[s])
            elif kind == BN_:
                for s in range(j, j + n):
                    parts = [staged[w][q][0][staged[w][q][1] == s] for q in (s - 1, s, s + 1) if q in staged[w]]
                    rec = np.concatenate(parts)
                    out[w][s] = rec[np.argsort(rec[:, 0], kind="stable")]
                    if w == W - 1:
                        push(out[w][s])
        if rank == 0:
            recv_until(ns - 1)
    for h in pending:
        h.wait()
    if rank == 0:
        final = np.concatenate([inb[j] for j in range(ns)])
        return final[np.argsort(final[:, 0])]
    return "ok"


@pytest.mark.parametrize("W,B,n_steps,calls", [(1, 2, 4, 1), (2, 2, 6, 2), (2, 3, 5, 1), (1, 3, 3, 2)])
def test_gloo_md_plan_emulation_equals_sequential(W, B, n_steps, calls):
    res = _spawn(_md_plan_worker, 2, W, B, n_steps, calls)
    final = res[0]
    g, x, v = _initial()
    xo, vo, Fo, _ = oracle.run(x, v, np.zeros_like(x), g.b, RC, DT, n_steps)
    assert np.array_equal(final[:, 0], np.arange(len(x)))
    d = final[:, 1:4] - xo
    d[:, 1:] -= g.b[1:] * np.round(d[:, 1:] / g.b[1:])
    assert np.max(np.abs(d)) < 1e-12
    assert np.max(np.abs(final[:, 4:7] - vo)) < 1e-11
