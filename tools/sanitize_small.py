"""Small circuits through every kernel family for compute-sanitizer (racecheck / memcheck):
group passes (c64, c128, several tile shapes), virtual-shard remaps, diag/cnot passes
(ONE_GATE), norm, gather and sampling.  n <= 16 so the sanitizer finishes in minutes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2008_00216_b200 as stv  # noqa: E402
from inputs import circuits as C  # noqa: E402

for dtype in ("c64", "c128"):
    for circ, kw in [(C.config(1), {}), (C.random_circuit(14, 200, 5), {}),
                     (C.qft_circuit(14, tail=100, seed=2), {}),
                     (C.random_circuit(13, 150, 7), dict(tile_bits=13, low_bits=5)),
                     (C.random_circuit(12, 120, 8), dict(flags=8))]:
        st = stv.State(circ.n, dtype)
        st.set_basis(circ.x0)
        st.apply(circ.gates, **kw)
        st.norm()
        st.amplitudes(np.arange(16, dtype=np.uint64))
        st.sample(64, seed=1)
        st.close()
    st = stv.State(14, dtype, virtual_g=2)
    st.apply(C.random_circuit(14, 120, 9).gates)
    st.norm()
    st.close()
print("sanitize_small done")
