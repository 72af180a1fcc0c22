import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, paper_2008_00216_b200 as stv
from inputs import circuits as C
def err(circ, dtype, **kw):
    st = stv.State(circ.n, dtype); st.set_basis(circ.x0); st.apply(circ.gates, **kw)
    psi = st.amplitudes(); s = st.stats(); st.close()
    r = oracle.compare(psi, oracle.run(circ))
    return r["max_abs"], {k: v for k, v in s["n_pass"].items() if v}
cases = [("qft22", C.qft_circuit(22, tail=200, seed=3)), ("qft12", C.qft_circuit(12, tail=200, seed=3)),
         ("qft12_notail", C.qft_circuit(12, tail=0, seed=3)), ("rand17", C.random_circuit(17, 300, 42)),
         ("cnots", C.random_circuit(14, 100, 5, kinds=["cnot", "h"])), ("diags", C.random_circuit(14, 100, 6, kinds=["cphase", "h", "t"]))]
for name, circ in cases:
    for dtype in ("c64", "c128"):
        for kw in (dict(), dict(flags=stv.OPT_NO_GROUPS), dict(budget=20), dict(budget=20, flags=stv.OPT_NO_GROUPS), dict(tile_bits=8, low_bits=3)):
            e, p = err(circ, dtype, **kw)
            print(f"{name:12s} {dtype} {str(kw):45s} err {e:.2e} {p}", flush=True)
