"""One-off full-state c3 parity (n=32): the GPU state (complex64, all 2^32 amplitudes)
against the complex128 oracle run gate by gate (64 GiB on the host; ~20 min on 16 cores).
Too slow for the round-end test budget; its result is committed in profiles/.
    python tools/c3_full_oracle.py [out.json]"""
import gc
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2008_00216_b200 as stv  # noqa: E402
from inputs import circuits as C  # noqa: E402

circ = C.config(3)
st = stv.State(circ.n, "c64")
st.set_basis(circ.x0)
st.apply(circ.gates)
stats = st.stats()
psi = st.read_state()                       # complex64, logical order, 32 GiB
norm = st.norm()
st.close()
import torch  # noqa: E402
gc.collect()
torch.cuda.empty_cache()
t0 = time.perf_counter()
ref = oracle.run(circ)                      # complex128, 64 GiB
t_or = time.perf_counter() - t0
r = oracle.compare(psi, ref, chunk=1 << 27)
line = {"test": "c3_c64_full_oracle", "n": circ.n, "gates": len(circ.gates), "max_abs": r["max_abs"],
        "fidelity": r["fidelity"], "norm_gpu": norm, "max_abs_rms": r["max_abs_rms"], "oracle_s": t_or,
        "cores": len(os.sched_getaffinity(0)), "passes": stats["n_pass"], "run_ms": stats["run_ms"],
        "bars": {"max_abs": 2e-6, "fidelity": 1 - 1e-5},
        "pass": bool(r["max_abs"] <= 2e-6 and r["fidelity"] >= 1 - 1e-5)}
print("PARITY", json.dumps(line), flush=True)
if len(sys.argv) > 1:
    json.dump(line, open(sys.argv[1], "w"), indent=1)
