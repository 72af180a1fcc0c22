"""A tiny CPU interpreter of the planner's PassList (tests only).

Executes the JSON plan returned by sv_plan_json (host code of the C-ABI
library) on a numpy complex128 state, op by op, with NO knowledge of the
gate table: it only sees fused matrices, diagonal phase forms (uint64
turns), CNOT ops, remaps and the final frame.  Comparing its output with the
oracle checks the planner's relabel frame, reordering, fusion, diagonal
clustering and remap bookkeeping (tier T0 planner) on CPU.
It shares no code with oracle/.
"""
import numpy as np

TWO64 = float(2 ** 64)


def _apply_dense(psi, n, tg, M):
    k = len(tg)
    t = psi.reshape([2] * n)
    axes = [n - 1 - b for b in reversed(tg)]
    t = np.moveaxis(t, axes, list(range(k)))
    shp = t.shape
    t = (M @ t.reshape(1 << k, -1)).reshape(shp)
    t = np.moveaxis(t, list(range(k)), axes)
    return np.ascontiguousarray(t).reshape(-1)


def _phase(n, op):
    j = np.arange(1 << n, dtype=np.uint64)
    ph = np.full(1 << n, np.uint64(int(op["cst"])), dtype=np.uint64)
    with np.errstate(over="ignore"):
        for b, a in op["lin"]:
            ph += ((j >> np.uint64(b)) & np.uint64(1)) * np.uint64(int(a))
        for p, q, a in op["quad"]:
            ph += ((j >> np.uint64(p)) & (j >> np.uint64(q)) & np.uint64(1)) * np.uint64(int(a))
    # exact turn -> angle: split the uint64 to keep 64-bit precision
    hi = (ph >> np.uint64(32)).astype(np.float64)
    lo = (ph & np.uint64(0xFFFFFFFF)).astype(np.float64)
    turns = (hi * 2.0 ** 32 + lo) / TWO64
    return np.exp(2j * np.pi * turns)


def _cnot(psi, n, c, t):
    j = np.arange(1 << n)
    sel = ((j >> c) & 1 == 1) & ((j >> t) & 1 == 0)
    a = j[sel]
    b = a | (1 << t)
    psi = psi.copy()
    psi[a], psi[b] = psi[b].copy(), psi[a].copy()
    return psi


def _bitswap(psi, n, a, b):
    j = np.arange(1 << n)
    src = j ^ ((((j >> a) ^ (j >> b)) & 1) * ((1 << a) | (1 << b)))
    return psi[src]


def _flat(ops):
    """Gate groups (type 4) are sequences of sub-ops applied in order."""
    for op in ops:
        if op["type"] == 4:
            yield from _flat(op["subs"])
        else:
            yield op


def run(plan, x0=0, psi=None):
    n = plan["n"]
    if psi is None:
        psi = np.zeros(1 << n, dtype=np.complex128)
        psi[x0] = 1
    psi = psi.astype(np.complex128)
    for ps in plan["passes"]:
        if ps["kind"] == 4:
            for gb, lb in ps["swaps"]:
                psi = _bitswap(psi, n, gb, lb)
            continue
        for op in _flat(ps["ops"]):
            if op["type"] == 1 and "sel" in op:
                # per-tile variants: the selector bits are untouched by the op, so each
                # selector value's subspace is invariant
                D = 1 << len(op["tg"])
                j = np.arange(1 << n)
                out = np.zeros_like(psi)
                for v, (vr, vi) in enumerate(zip(op["vre"], op["vim"])):
                    M = (np.array(vr) + 1j * np.array(vi)).reshape(D, D)
                    m = np.ones(1 << n, dtype=bool)
                    for i, b in enumerate(op["sel"]):
                        m &= ((j >> b) & 1) == ((v >> i) & 1)
                    out[m] = _apply_dense(psi, n, op["tg"], M)[m]
                psi = out
            elif op["type"] == 1:
                D = 1 << len(op["tg"])
                M = (np.array(op["re"]) + 1j * np.array(op["im"])).reshape(D, D)
                psi = _apply_dense(psi, n, op["tg"], M)
            elif op["type"] == 2:
                psi = psi * _phase(n, op)
            else:
                psi = _cnot(psi, n, op["c"], op["t"])
    return psi


def logical(plan, psi):
    """Read the physical state in logical order through the final frame."""
    n = plan["n"]
    perm = plan["perm"]
    xm = int(plan["xmask"])
    j = np.arange(1 << n)
    p = np.zeros(1 << n, dtype=np.int64)
    for q in range(n):
        p |= ((j >> q) & 1) << perm[q]
    return psi[p ^ xm]
