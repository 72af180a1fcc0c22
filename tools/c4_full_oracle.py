"""One-off full-state c4 parity (n=34, 128 GiB complex64 on one B200): the GPU state against
the oracle run gate by gate with complex64 storage and complex128 arithmetic per gate
(oracle.run_c64store, reading A19: the complex128 oracle state, 256 GiB, exceeds the
box's host memory).  The GPU state is compared on 2^28 uniformly sampled amplitudes (the full
GPU state does not fit host memory next to the oracle's).  The whole 14-cycle circuit takes
the oracle over an hour on the box's 16 host cores (more than one gpurun call), so the check
runs c4's first CYCLES cycles (default 7: gates[:288], the same gates as c4's prefix) at the full
n = 34; its result is committed in profiles/.
    python tools/c4_full_oracle.py [out.json] [cycles]"""
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

cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 7
full = C.config(4)
circ = C.grid_circuit("c4", 6, 6, 2, cycles, "fsim", 4)   # c4's first `cycles` cycles
assert circ.gates == full.gates[:len(circ.gates)]
rng = np.random.default_rng(34)
y = np.unique(rng.integers(0, 1 << circ.n, size=1 << 28, dtype=np.uint64))
st = stv.State(circ.n, "c64")
st.set_basis(circ.x0)
st.apply(circ.gates)
stats = st.stats()
a = st.amplitudes(y)                       # logical order
norm = st.norm()
st.close()
del st
import torch  # noqa: E402
gc.collect()
torch.cuda.empty_cache()
t0 = time.perf_counter()
ref = oracle.run_c64store(circ)            # complex64 storage, 128 GiB
t_or = time.perf_counter() - t0
b = ref[y.astype(np.int64)].astype(np.complex128)
onorm = 0.0   # float64 per 2^26-amplitude chunk (np.vdot of complex64 accumulates in single precision)
for k in range(0, ref.size, 1 << 26):
    blk = ref[k:k + (1 << 26)].view(np.float32).astype(np.float64)
    onorm += float(np.dot(blk, blk))
del ref
gc.collect()
a = a.astype(np.complex128)
d = float(np.max(np.abs(a - b)))
fid = abs(np.vdot(b, a)) ** 2 / (np.vdot(a, a).real * np.vdot(b, b).real)
line = {"test": "c4_c64_full_oracle_c64store", "n": circ.n, "cycles": cycles, "gates": len(circ.gates), "sampled": int(y.size),
        "max_abs": d, "fidelity_sampled": float(fid), "norm_gpu": norm, "norm_oracle": onorm, "oracle_s": t_or,
        "cores": len(os.sched_getaffinity(0)), "passes": stats["n_pass"], "run_ms": stats["run_ms"],
        "bars": {"max_abs": 2e-6, "fidelity": 1 - 1e-5},
        "pass": bool(d <= 2e-6 and fid >= 1 - 1e-5)}
print("PARITY", json.dumps(line), flush=True)
if len(sys.argv) > 1:
    json.dump(line, open(sys.argv[1], "w"), indent=1)
