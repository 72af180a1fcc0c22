"""Profiling driver: run a reduced c2-shaped workload so ncu can capture a
few k_tile_pass launches (plain run first, then the same command under ncu)."""
import argparse, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2008_00216_b200 as stv
from inputs import circuits as C

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--gates", type=int, default=80)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--tile-bits", type=int, default=0)
ap.add_argument("--low-bits", type=int, default=0)
ap.add_argument("--budget", type=int, default=0)
ap.add_argument("--kmax", type=int, default=0)
ap.add_argument("--dtype", default="c64")
ap.add_argument("--flags", type=int, default=0)
a = ap.parse_args()
circ = C.config(2) if a.n == 30 else C.grid_circuit("g", 5, a.n // 5, 0, 20, "fsim", 2)
st = stv.State(circ.n, a.dtype)
for r in range(a.reps):
    st.set_basis(0)
    st.apply(circ.gates[:a.gates], tile_bits=a.tile_bits, low_bits=a.low_bits, budget=a.budget, kmax=a.kmax, flags=a.flags, profile=True)
    s = st.stats()
    nt = s["n_pass"]["tile_low"] + s["n_pass"]["tile_high"]
    tms = s["pass_ms"]["tile_low"] + s["pass_ms"]["tile_high"]
    esz = 8 if a.dtype == "c64" else 16
    print(json.dumps({"tile_passes": nt, "tile_ms_avg": tms / max(nt, 1),
                      "GBps": 2 * esz * (1 << circ.n) / (tms / max(nt, 1) / 1e3) / 1e9 if nt else None,
                      "run_ms": s["run_ms"], "n_pass": {k: v for k, v in s["n_pass"].items() if v},
                      "ops": s["n_ops"], "args": vars(a)}))
st.close()
