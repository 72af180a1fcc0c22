"""GPU fuzz (not part of the test suite): seeded circuits at n = 20..24 -- full 12-bit tiles, so
complex64 runs on the tensor-core pass -- with planner options, dtype and virtual shards drawn
per case, each compared element-wise with the CPU oracle (bars of tests/test_gpu_parity.py).
    python tools/gpu_fuzz.py [seconds=480] [out.jsonl] [nmin=20] [nmax=24]
Prints one JSON line per case and a summary; exit code 1 if any case fails."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (a checker: this tool is test infrastructure)
import paper_2008_00216_b200 as stv  # noqa: E402
from inputs import circuits as C  # noqa: E402
from inputs.circuits import SplitMix64  # noqa: E402

budget_s = float(sys.argv[1]) if len(sys.argv) > 1 else 480.0
out = open(sys.argv[2], "w") if len(sys.argv) > 2 else None
nmin = int(sys.argv[3]) if len(sys.argv) > 3 else 20
nmax = int(sys.argv[4]) if len(sys.argv) > 4 else 24
OPTS = [dict(), dict(), dict(kmax=1), dict(kmax=2), dict(kmax=3), dict(low_bits=5), dict(low_bits=6),
        dict(low_bits=7), dict(budget=400), dict(budget=3000), dict(flags=2), dict(flags=4), dict(flags=16),
        dict(flags=128), dict(flags=0x400), dict(flags=0x800), dict(tile_bits=11), dict(tile_bits=13),
        dict(kmax=2, low_bits=5), dict(kmax=3, budget=400), dict(kmax=2, flags=0x800)]
KINDS = [None, None, ["h", "cz", "t", "x", "cnot"], ["u1", "fsim"], ["u2", "cphase", "h"], ["cnot", "x", "cz", "t", "h"]]
TOL = {"c64": 2e-6, "c128": 1e-12}
rng = SplitMix64(20260101 + 1000 * nmin + nmax)
t0 = time.time()
ncase = nfail = 0
while time.time() - t0 < budget_s:
    n = nmin + rng.u(nmax - nmin + 1)
    shape = rng.u(4)
    seed = 1000 * (nmin - 19) + ncase
    if shape == 0:
        circ = C.qft_circuit(n, 60 + rng.u(100), seed, "fz")
    elif shape == 1:
        R = 4 if n % 4 == 0 else 5 if n % 5 == 0 else 3 if n % 3 == 0 else 2
        if n % R:
            circ = C.random_circuit(n, 200 + rng.u(300), seed)
        else:
            circ = C.grid_circuit("fz", R, n // R, 0, 6 + rng.u(8), "fsim" if rng.u(2) else "cz", seed)
    else:
        circ = C.random_circuit(n, 150 + rng.u(350), seed, KINDS[rng.u(len(KINDS))])
    kw = OPTS[rng.u(len(OPTS))]
    dtype = "c128" if rng.u(4) == 0 else "c64"
    g = (0, 0, 1, 2, 3)[rng.u(5)]
    rec = {"case": ncase, "circuit": circ.name, "n": circ.n, "gates": len(circ.gates), "opts": kw, "dtype": dtype, "g": g}
    try:
        st = stv.State(circ.n, dtype, virtual_g=g) if g else stv.State(circ.n, dtype)
        st.set_basis(circ.x0)
        st.apply(circ.gates, **kw)
        s = st.stats()
        psi = st.amplitudes()
        st.close()
        r = oracle.compare(psi, oracle.run(circ))
        ok = r["max_abs"] <= TOL[dtype] and (dtype == "c128" or r["fidelity"] >= 1 - 1e-5)
        rec.update(max_abs=r["max_abs"], fidelity=r["fidelity"], tc_passes=s.get("n_tc_pass"), ok=bool(ok))
    except Exception as e:  # a refused launch is a failure too
        rec.update(error=str(e), ok=False)
    ncase += 1
    nfail += not rec["ok"]
    line = json.dumps(rec, default=float)
    print(line, flush=True)
    if out:
        out.write(line + "\n")
        out.flush()
print(json.dumps({"cases": ncase, "failed": nfail, "seconds": round(time.time() - t0, 1)}))
sys.exit(1 if nfail else 0)
