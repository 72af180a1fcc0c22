"""Per-pass device times of one config in several planner modes (STV_PASS_LOG), e.g.
    python tools/pass_times.py c2 0 256      # default (tensor-core passes) vs SV_OPT_NO_TC
Prints one row per pass: groups, M steps, FMA flops/amp and ms per mode."""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_00216_b200 as stv  # noqa: E402
from inputs import circuits as C  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
modes = [int(x) for x in sys.argv[2:]] or [0, 256]
circ = C.config(int(cfg[1:]))
res = {}
for flags in modes:
    st = stv.State(circ.n, "c64")
    for rep in range(3):
        log = tempfile.mktemp()
        os.environ["STV_PASS_LOG"] = log
        st.set_basis(circ.x0)
        st.apply(circ.gates, flags=flags, profile=True)
    res[flags] = [json.loads(line) for line in open(log)]
    st.close()
print("pass groups msteps flops/amp " + " ".join("ms[%d]" % f for f in modes))
for i, p in enumerate(res[modes[0]]):
    print("%4d %6d %6d %9.0f " % (i, p["groups"], p["msteps"], p["flops_per_amp"]) +
          " ".join("%7.3f" % res[f][i]["ms"] for f in modes))
print("sum", " ".join("%.2f" % sum(p["ms"] for p in res[f]) for f in modes))
