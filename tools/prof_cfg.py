"""Run one config's circuit once (for ncu captures of its passes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401
import paper_2008_00216_b200 as stv
from inputs import circuits as C
circ = C.config(int(sys.argv[1]))
st = stv.State(circ.n, "c64")
st.set_basis(circ.x0)
st.apply(circ.gates, profile=True)
s = st.stats()
print({k: v for k, v in s["n_pass"].items() if v}, s["run_ms"], s["pass_ms"])
