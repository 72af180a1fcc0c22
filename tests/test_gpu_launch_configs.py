"""Parity of the non-default k_group_pass launch configurations (-m gpu).

`STV_GCFG` (csrc/kernels.cu launch_group_pass) selects, once per process, the
group-pass instantiation: 0 = one tile buffer at 4 CTAs/SM (default),
1 = 128 threads x 2 register vectors, 2 = 3-stage ring, 3 = 2-stage ring at
3 CTAs/SM.  Each configuration runs in its own process against the CPU oracle
(same bars as test_gpu_parity.py: c64 max|delta| <= 2e-6, F >= 1 - 1e-5).
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import torch
import oracle
from inputs import circuits as C
import paper_2008_00216_b200 as stv
out = []
for circ in (C.random_circuit(14, 200, 11), C.config(1), C.qft_circuit(13, 40, 5)):
    st = stv.State(circ.n, "c64")
    st.set_basis(circ.x0)
    st.apply(circ.gates)
    psi = st.amplitudes()
    st.close()
    r = oracle.compare(psi, oracle.run(circ))
    out.append([float(r["max_abs"]), float(r["fidelity"])])
print(json.dumps(out))
"""


@pytest.mark.parametrize("cfg", ["0", "1", "2", "3"])
def test_group_pass_launch_config_parity(cfg):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, STV_GCFG=cfg)
    p = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    for max_abs, fid in json.loads(p.stdout.strip().splitlines()[-1]):
        assert max_abs <= 2e-6 and fid >= 1 - 1e-5, (cfg, max_abs, fid)


def test_tc_pass_small_tiles_parity():
    """STV_TC_SMALL=1: the tensor-core pass also on tiles of fewer than 12 bits (by default
    those run on the CUDA-core pass): its non-full-tile variant (threads beyond the tile's
    vectors idle) against the oracle on the small circuits above."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, STV_TC_SMALL="1")
    p = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    for max_abs, fid in json.loads(p.stdout.strip().splitlines()[-1]):
        assert max_abs <= 2e-6 and fid >= 1 - 1e-5, (max_abs, fid)
