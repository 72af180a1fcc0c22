"""Multi-process CPU tests of the N>1 path's host logic (gloo, world_size 2
and 4, 127.0.0.1; -m "not gpu").

Each rank holds the 2^{n-g} amplitudes whose top g physical bits equal its
rank.  A distributed CPU interpreter executes the plan the
library produces for n_global = g: ops act on local bits, diagonal phases
and CNOT controls on global bits are evaluated from the rank, and every
remap is the all-to-all of csrc/api.cpp `dist_remap` -- chunk c (the value
of the swapped local bits, ordered by global bit) goes to
sv_remap_peers(...)[c] and the chunk received from that peer lands in slot c
-- done with torch.distributed send/recv over gloo.  The gathered state,
read through the final frame, must equal the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2008_00216_b200 as stv
from inputs import circuits as C
from tests import plan_interp as PI


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _insert_bits(k, positions_bits):
    """Insert fixed bits (pos, value), ascending pos, into integer array k."""
    i = k.copy()
    for p, v in sorted(positions_bits):
        i = ((i >> p) << (p + 1)) | (v << p) | (i & ((1 << p) - 1))
    return i


def _remap(shard, nl, g, rank, swaps):
    sw = sorted(swaps)                      # chunk bit i <-> i-th swap ordered by global bit
    m = len(sw)
    gbits = 0
    for gb, _ in sw:
        gbits |= 1 << (gb - nl)
    peers = stv.remap_peers(g, rank, gbits, m)
    mine = sum(((rank >> (gb - nl)) & 1) << i for i, (gb, _) in enumerate(sw))
    k = np.arange(1 << (nl - m))
    new = shard.copy()
    reqs = []
    recv = {}
    for c in range(1 << m):
        if c == mine:
            continue
        idx = _insert_bits(k, [(lb, (c >> i) & 1) for i, (_, lb) in enumerate(sw)])
        out = torch.from_numpy(np.ascontiguousarray(shard[idx]).view(np.float64).copy())
        inn = torch.empty_like(out)
        # lower rank sends first: deadlock-free pairwise exchange
        if rank < peers[c]:
            dist.send(out, peers[c]); dist.recv(inn, peers[c])
        else:
            dist.recv(inn, peers[c]); dist.send(out, peers[c])
        new[idx] = inn.numpy().view(np.complex128)
    return new


def _run_dist(rank, world, port, n, seed, tile_bits, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = world.bit_length() - 1
        nl = n - g
        circ = C.random_circuit(n, 160, seed)
        plan = stv.plan_json(n, circ.gates, n_global=g, tile_bits=tile_bits, low_bits=2)
        shard = np.zeros(1 << nl, dtype=np.complex128)
        if (circ.x0 >> nl) == rank:
            shard[circ.x0 & ((1 << nl) - 1)] = 1
        jl = np.arange(1 << nl, dtype=np.uint64)
        full_j = jl | np.uint64(rank << nl)
        nremap = 0
        for ps in plan["passes"]:
            if ps["kind"] == 4:
                shard = _remap(shard, nl, g, rank, [tuple(s) for s in ps["swaps"]])
                nremap += 1
                continue
            for op in PI._flat(ps["ops"]):
                if op["type"] == 1 and "sel" in op:
                    # per-tile variants selected by bits outside the tile (global bits: this rank's)
                    assert max(op["tg"]) < nl
                    D = 1 << len(op["tg"])
                    out = np.zeros_like(shard)
                    for v, (vr, vi) in enumerate(zip(op["vre"], op["vim"])):
                        M = (np.array(vr) + 1j * np.array(vi)).reshape(D, D)
                        m = np.ones(1 << nl, dtype=bool)
                        for i, b in enumerate(op["sel"]):
                            m &= ((full_j >> np.uint64(b)) & np.uint64(1)) == np.uint64((v >> i) & 1)
                        out[m] = PI._apply_dense(shard, nl, op["tg"], M)[m]
                    shard = out
                elif op["type"] == 1:
                    assert max(op["tg"]) < nl
                    D = 1 << len(op["tg"])
                    M = (np.array(op["re"]) + 1j * np.array(op["im"])).reshape(D, D)
                    shard = PI._apply_dense(shard, nl, op["tg"], M)
                elif op["type"] == 2:
                    # phase form over FULL indices: global bits come from the rank
                    ph = np.full(1 << nl, np.uint64(int(op["cst"])), dtype=np.uint64)
                    with np.errstate(over="ignore"):
                        for b, a in op["lin"]:
                            ph += ((full_j >> np.uint64(b)) & np.uint64(1)) * np.uint64(int(a))
                        for p, r, a in op["quad"]:
                            ph += ((full_j >> np.uint64(p)) & (full_j >> np.uint64(r)) & np.uint64(1)) * np.uint64(int(a))
                    hi = (ph >> np.uint64(32)).astype(np.float64)
                    lo = (ph & np.uint64(0xFFFFFFFF)).astype(np.float64)
                    shard = shard * np.exp(2j * np.pi * (hi * 2.0 ** 32 + lo) / 2.0 ** 64)
                else:
                    c, t = op["c"], op["t"]
                    assert t < nl
                    if c >= nl:                # control on a global bit: per-rank predicate
                        if (rank >> (c - nl)) & 1:
                            shard = shard[np.arange(1 << nl) ^ (1 << t)]
                    else:
                        shard = PI._cnot(shard, nl, c, t)
        parts = [torch.empty(2 << nl, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(shard.view(np.float64).copy()))
        if rank == 0:
            full = np.concatenate([p.numpy().view(np.complex128) for p in parts])
            psi = PI.logical(plan, full)
            ref = oracle.run(circ)
            q.put((float(np.max(np.abs(psi - ref))), nremap))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,seed,tile_bits", [(2, 9, 1, 5), (2, 10, 2, 6), (4, 10, 3, 5)])
def test_distributed_plan_with_remaps(world, n, seed, tile_bits):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_dist, args=(r, world, port, n, seed, tile_bits, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    err, nremap = q.get(timeout=5)
    assert nremap > 0
    assert err < 1e-11
