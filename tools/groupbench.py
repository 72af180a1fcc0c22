"""Marginal cost of gate-group sub-ops in k_group_pass (one pass, n=30 c64).

Circuits of m random 2-qubit unitaries on rotating overlapping pairs of 4
qubits (so they stay separate U2 sub-ops of one group), optionally with a
controlled-phase to a qubit outside the group after each (a DIAG sub-op with a
per-tile table).  Prints ms per pass, marginal ns per U2, and the FMA-pipe
fraction of that marginal cost (8 FFMA2 x 2 cycles per amplitude per U2)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch  # noqa: F401
import paper_2008_00216_b200 as stv

n = int(os.environ.get("GB_N", "30"))
st = stv.State(n, "c64")
rng = np.random.default_rng(1)


def rand_u(d):
    z = rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d))
    q, r = np.linalg.qr(z)
    q = q * (np.diag(r) / np.abs(np.diag(r)))
    return [v for c in q.reshape(-1) for v in (c.real, c.imag)]


def circuit(m, diag, qs=(4, 5, 6, 7)):
    """diag: None; 'out' = controlled phase to a qubit outside the tile (folds into per-tile
    variant matrices); 'v' = to an in-tile qubit outside the group (a per-tile table sub-op)."""
    pairs = [(qs[0], qs[1]), (qs[1], qs[2]), (qs[2], qs[3]), (qs[3], qs[0])]
    g = []
    if diag == "v":   # dense gates pull the partner qubits into the tile (V-bits of the group)
        g += [("h", (9,), ()), ("h", (10,), ()), ("h", (11,), ())]
    for i in range(m):
        g.append(("u2", pairs[i % 4], rand_u(4)))
        if diag == "out":
            g.append(("cphase", (pairs[i % 4][0], 20 + i % 5), ((1, 6),)))
        elif diag == "v":
            g.append(("cphase", (pairs[i % 4][0], 9 + i % 3), ((1, 6),)))
    return g


def run(gates, reps=3):
    best = None
    for _ in range(reps):
        st.apply(gates, budget=100000, tile_bits=12, profile=True)
        s = st.stats()
        ms = s["pass_ms"]["tile_low"] + s["pass_ms"]["tile_high"]
        best = ms if best is None else min(best, ms)
    return best, s["n_pass"], s["n_ops"]


out = {}
for diag in (None, "out", "v"):
    pts = {}
    for m in (4, 16, 48):
        ms, npass, ops = run(circuit(m, diag))
        pts[m] = ms
        out[f"u2{diag or ''}_m{m}"] = {"ms": ms, "passes": npass, "ops": ops}
    per = (pts[48] - pts[16]) / 32
    fma_ms = 8 * 2 * 2 ** n / (148 * 4 * 32 * 1.965e9) * 1e3   # 8 FFMA2/amp, 2 cycles per warp FFMA2
    out[f"u2{diag or ''}_per_u2_ms"] = per
    out[f"u2{diag or ''}_fma_fraction"] = fma_ms / per
print(json.dumps(out, indent=1))
