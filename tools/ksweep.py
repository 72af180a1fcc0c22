"""c2 fusion k-sweep: for k = kmax = 1..6 the
register bits of a gate group (the fused dense block), on the tensor-core path and on the
CUDA-core FMA path (SV_OPT_NO_TC): passes, groups, FMA flops/amp per pass, tensor-core
operator steps, sec/circuit and the per-pass HBM GB/s.  k = 5, 6 exceed the 16-amplitude
register vector of a group and are clamped to 4 by the library (reported as such).
    python tools/ksweep.py [out.md]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2008_00216_b200 as stv  # noqa: E402
from inputs import circuits as C  # noqa: E402

circ = C.config(2)
n = circ.n
rows = []
st = stv.State(n, "c64")
arr, keep = stv.marshal(circ.gates)
for k in range(1, 7):
    for flags, path in ((0, "tensor-core"), (256, "FMA")):
        o = stv.options(kmax=k, flags=flags, profile=True)
        times = []
        for rep in range(4):
            st.set_basis(0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st.apply_marshalled(arr, len(circ.gates), o)
            e1.record()
            torch.cuda.synchronize()
            if rep:
                times.append(e0.elapsed_time(e1))
        s = st.stats()
        npass = s["n_pass"]["tile_low"] + s["n_pass"]["tile_high"]
        tile_ms = s["pass_ms"]["tile_low"] + s["pass_ms"]["tile_high"]
        plan = stv.plan_json(n, circ.gates, kmax=k, flags=flags)
        groups = sum(len(p["ops"]) for p in plan["passes"])
        r = {"k": k, "k_effective": min(k, 4), "path": path, "passes": npass, "groups": groups,
             "tc_steps": s["n_tc_steps"], "fma_flops_per_amp_per_pass": s["alg_flops"] / (1 << n) / max(1, npass),
             "sec_per_circuit": min(times) / 1e3,
             "pass_gbs": npass * 16 * (1 << n) / (tile_ms / 1e3) / 1e9 if tile_ms else None}
        rows.append(r)
        print(json.dumps(r), flush=True)
st.close()
out = sys.argv[1] if len(sys.argv) > 1 else None
if out:
    with open(out, "w") as f:
        f.write("# c2 fusion k-sweep (n=30, complex64, one B200)\n\n")
        f.write("k = register bits of a gate group (the fused dense block). k = 5, 6 are clamped to 4.\n\n")
        f.write("| k | path | passes | groups | TC operator steps | FMA flop/amp/pass | per-pass GB/s | sec/circuit |\n")
        f.write("|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write("| %d%s | %s | %d | %d | %d | %.0f | %.0f | %.4f |\n" % (
                r["k"], "" if r["k"] <= 4 else " (=4)", r["path"], r["passes"], r["groups"], r["tc_steps"],
                r["fma_flops_per_amp_per_pass"], r["pass_gbs"] or 0, r["sec_per_circuit"]))
