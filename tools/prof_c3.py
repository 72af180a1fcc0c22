import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_00216_b200 as stv
from inputs import circuits as C
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
circ = C.qft_circuit(n, 200, 3)
st = stv.State(n)
st.set_basis(circ.x0); st.apply(circ.gates, profile=True); s = st.stats()
print({k: v for k, v in s["n_pass"].items() if v}, s["run_ms"], s["n_ops"], s["alg_flops"] / 1e12)
p = stv.plan_json(n, circ.gates)
for ps in p["passes"]:
    subs = [so for o in ps["ops"] if o["type"] == 4 for so in o["subs"]]
    nd = sum(1 for so in subs if so["type"] == 2)
    terms = sum(len(so["lin"]) + len(so["quad"]) for so in subs if so["type"] == 2)
    print("pass groups", len(ps["ops"]), "subs", len(subs), "diag subs", nd, "diag terms", terms)
