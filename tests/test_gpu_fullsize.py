"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (default planner options), -m gpu.

c2 (n=30): element-by-element against the full complex128 oracle (16 GiB;
the GPU box has 196 GB of host RAM).  c3 (n=32): the phase-state invariant
|psi_y| = 2^-16 on every amplitude after the tail (permutations + phases),
and the QFT closed form on 2^20 sampled amplitudes before the tail.  c4
(n=34, 128 GiB complex64 on one B200): mirror test C^dagger C |0> = |0>
and the norm -- properties that hold at any size.
"""
import gc
import math

import numpy as np
import pytest

import oracle
from inputs import circuits as C

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def stv():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2008_00216_b200 as m
    m.lib()
    return m


def _free():
    import torch
    gc.collect()
    torch.cuda.empty_cache()


def test_c2_full_parity(stv):
    circ = C.config(2)
    st = stv.State(circ.n, "c64")
    st.set_basis(circ.x0)
    st.apply(circ.gates)
    psi = st.read_state()                 # complex64, logical order, 8 GiB
    norm = st.norm()
    st.close()
    _free()
    ref = oracle.run(circ)                # complex128, 16 GiB, all host cores
    r = oracle.compare(psi, ref, chunk=1 << 27)
    del ref, psi
    assert r["max_abs"] <= 2e-6, r
    assert r["fidelity"] >= 1 - 1e-5, r
    assert abs(norm - 1) < 1e-4


def test_c3_full_invariants(stv):
    circ = C.config(3)
    n = circ.n
    nq = len(C.qft_gates(n))
    st = stv.State(n, "c64")
    st.set_basis(circ.x0)
    st.apply(circ.gates[:nq])             # QFT of |x0>
    rng = np.random.default_rng(3)
    y = np.unique(rng.integers(0, 1 << n, size=1 << 20, dtype=np.uint64))
    got = st.amplitudes(y)
    ref = 2 ** (-n / 2) * np.exp(2j * np.pi * ((circ.x0 * y.astype(object)) % (1 << n)).astype(np.float64) / (1 << n))
    assert np.max(np.abs(got - ref)) <= 2e-6
    st.apply(circ.gates[nq:])             # + 200 CNOT/X/CZ/T
    chunk = 1 << 28
    worst = 0.0
    for first in range(0, 1 << n, chunk):
        a = st.read_state(first, chunk)
        worst = max(worst, float(np.max(np.abs(np.abs(a) - 2.0 ** -16))))
    norm = st.norm()
    st.close()
    _free()
    assert worst <= 2e-6 and abs(norm - 1) < 1e-4


def test_c4_mirror_and_norm(stv):
    import torch
    free, _ = torch.cuda.mem_get_info()
    if free < (8 << 34) + (4 << 30):
        pytest.skip("needs a 180 GB B200 (128 GiB state)")
    circ = C.config(4)
    st = stv.State(circ.n, "c64")
    st.set_basis(0)
    st.apply(circ.gates)
    norm = st.norm()
    st.apply(C.inverse_gates(circ.gates))
    a0 = st.amplitudes(np.array([0, 1, (1 << 34) - 1], dtype=np.uint64))
    st.close()
    _free()
    assert abs(norm - 1) < 1e-4
    assert abs(a0[0]) ** 2 >= 1 - 1e-5 and abs(a0[1]) < 1e-4 and abs(a0[2]) < 1e-4
