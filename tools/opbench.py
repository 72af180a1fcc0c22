"""Per-op cost of the fused tile pass: single-pass circuits with m ops of one
kind (dense k=1..4, diag, cnot) on a 2^30 c64 state; prints ms per pass and
the marginal cost per op in ns and in 'instruction-equivalents per amplitude'
(148 SMs x 4 issue x 32 lanes x 1.965 GHz)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2008_00216_b200 as stv

n = int(os.environ.get("OPB_N", "30"))
dtype = os.environ.get("OPB_DT", "c64")
st = stv.State(n, dtype)
IPS = 148 * 4 * 32 * 1.965e9

def run(gates, kmax, reps=3):
    best = None
    for _ in range(reps):
        st.apply(gates, kmax=kmax, budget=100000, tile_bits=12, profile=True)
        s = st.stats()
        tiles = s["n_pass"]["tile_low"] + s["n_pass"]["tile_high"]
        ms = s["pass_ms"]["tile_low"] + s["pass_ms"]["tile_high"]
        best = ms if best is None else min(best, ms)
    return best, tiles, s["n_ops"]

def gates_for(kind, m):
    g = []
    if kind == "k1":
        for i in range(m): g.append(("sx" if i % 2 else "sy", (i % 11,), ()))
    elif kind in ("k2", "k3", "k4"):
        k = int(kind[1])
        for i in range(m):
            # ops on rotating disjoint groups: consecutive groups overlap in one qubit,
            # so they cannot merge into one op but stay in one pass
            base = (i * (k - 1)) % (12 - k)
            for q in range(k): g.append(("sx" if (i + q) % 2 else "sy", (base + q,), ()))
            g.append(("cz", (base, base + k - 1), ()))
    elif kind == "diag":
        for i in range(m):
            g.append(("sx", (i % 11,), ()))
            g.append(("cphase", (i % 11, 20 + i % 7), ((1, 7),)))
    elif kind == "cnot":
        for i in range(m): g.append(("cnot", (20 + i % 5, i % 11), ()))
    return g

res = {}
base, _, _ = run([("sx", (0,), ())], 1)
res["one_k1_op"] = base
for kind, kmax in [("k1", 1), ("k2", 2), ("k3", 3), ("k4", 4), ("diag", 1), ("cnot", 1)]:
    for m in (4, 8):
        ms, tiles, ops = run(gates_for(kind, m), kmax)
        res[f"{kind}_m{m}"] = {"ms": ms, "passes": tiles, "ops": ops}
    a = res[f"{kind}_m4"]; b = res[f"{kind}_m8"]
    nops = (b["ops"]["dense"] + b["ops"]["diag"] + b["ops"]["cnot"]) - (a["ops"]["dense"] + a["ops"]["diag"] + a["ops"]["cnot"])
    if a["passes"] == b["passes"] == 1 and nops > 0:
        per = (b["ms"] - a["ms"]) / nops
        res[f"{kind}_per_op_ms"] = per
        res[f"{kind}_instr_per_amp"] = per / 1e3 * IPS / 2 ** n
print(json.dumps(res, indent=1))
