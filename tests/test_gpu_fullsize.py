"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (default planner options), -m gpu.  Every test prints (and appends to
$STV_PARITY_LOG, one JSON line each, if set) max |delta|, the fidelity and the
norm it measured, so profiles/r02_parity.md and BASELINE.md section 5 are
filled from the run itself.

c2 (n=30): element by element against the full complex128 oracle (16 GiB on
the host), in complex64 (bar 2e-6, F >= 1 - 1e-5), in complex128 (bar 1e-12),
and through virtual shards with g = 3 global qubits (the sharded path, 8
shards, bar 2e-6).
c3 (n=32): every amplitude against the phase-state invariant |psi_y| = 2^-16,
and 2^20 sampled amplitudes element by element against the oracle's
single-amplitude paths (QFT closed form, then the CNOT/X/CZ/T tail one row at a
time: oracle.monomial_amplitudes) -- the full 64 GiB oracle takes longer than
the test budget on the 16 host cores.
c4 (n=34, 128 GiB complex64 on one B200): SURVEY.md 8(c) proxies -- the G=1
run and virtual shards g=1 and g=2 agree on 2^26 sampled amplitudes (2e-6),
mirror test C^dagger C |0> = |0>, norm.
"""
import gc
import json
import os

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


def record(name, **vals):
    line = {"test": name, **{k: (float(v) if isinstance(v, (np.floating, float)) else v) for k, v in vals.items()}}
    print("PARITY", json.dumps(line))
    path = os.environ.get("STV_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(line) + "\n")


@pytest.fixture(scope="module")
def c2_ref():
    circ = C.config(2)
    import time
    t0 = time.perf_counter()
    ref = oracle.run(circ)                # complex128, 16 GiB, all host cores
    record("c2_oracle", n=circ.n, gates=len(circ.gates), oracle_s=time.perf_counter() - t0,
           cores=len(os.sched_getaffinity(0)))
    yield circ, ref
    del ref
    gc.collect()


def _run_full(stv, circ, dtype, **kw):
    st = stv.State(circ.n, dtype, **kw)
    st.set_basis(circ.x0)
    st.apply(circ.gates)
    stats = st.stats()
    psi = st.read_state()                 # native dtype, logical order
    norm = st.norm()
    st.close()
    _free()
    return psi, norm, stats


@pytest.mark.parametrize("dtype,bar", [("c64", 2e-6), ("c128", 1e-12)])
def test_c2_full_parity(stv, c2_ref, dtype, bar):
    circ, ref = c2_ref
    psi, norm, stats = _run_full(stv, circ, dtype)
    r = oracle.compare(psi, ref, chunk=1 << 27)
    del psi
    record(f"c2_{dtype}", n=circ.n, max_abs=r["max_abs"], fidelity=r["fidelity"], norm=norm,
           max_abs_rms=r["max_abs_rms"], passes=stats["n_pass"], run_ms=stats["run_ms"])
    assert r["max_abs"] <= bar, r
    assert r["fidelity"] >= 1 - 1e-5, r
    assert abs(norm - 1) < (1e-4 if dtype == "c64" else 1e-12)


def test_c2_virtual_g3_vs_oracle(stv, c2_ref):
    circ, ref = c2_ref
    psi, norm, stats = _run_full(stv, circ, "c64", virtual_g=3)
    r = oracle.compare(psi, ref, chunk=1 << 27)
    del psi
    record("c2_c64_virtual_g3", n=circ.n, max_abs=r["max_abs"], fidelity=r["fidelity"], norm=norm,
           remaps=stats["n_pass"]["remap"], remap_bytes=stats["remap_bytes"])
    assert r["max_abs"] <= 2e-6 and r["fidelity"] >= 1 - 1e-5, r
    assert stats["n_pass"]["remap"] > 0


def test_c3_full(stv):
    circ = C.config(3)
    n = circ.n
    nq = len(C.qft_gates(n))
    st = stv.State(n, "c64")
    st.set_basis(circ.x0)
    st.apply(circ.gates)
    rng = np.random.default_rng(3)
    y = np.unique(rng.integers(0, 1 << n, size=1 << 20, dtype=np.uint64))
    got = st.amplitudes(y)
    worst = 0.0                             # phase-state invariant on every amplitude
    chunk = 1 << 28
    for first in range(0, 1 << n, chunk):
        a = st.read_state(first, chunk)
        worst = max(worst, float(np.max(np.abs(np.abs(a) - 2.0 ** -16))))
    norm = st.norm()
    st.close()
    _free()
    ref = oracle.monomial_amplitudes(n, circ.gates[nq:], lambda x: oracle.qft_basis_amplitudes(n, circ.x0, x), y)
    d = float(np.max(np.abs(got - ref)))
    ov = np.vdot(ref, got)
    fid = abs(ov) ** 2 / (np.vdot(ref, ref).real * np.vdot(got, got).real)
    record("c3_c64", n=n, sampled=int(y.size), max_abs=d, fidelity_sampled=fid, invariant_max_dev=worst, norm=norm)
    assert d <= 2e-6 and fid >= 1 - 1e-5
    assert worst <= 2e-6 and abs(norm - 1) < 1e-4


def _big_gpu(need_bytes):
    import torch
    free, _ = torch.cuda.mem_get_info()
    return free >= need_bytes


def test_c4_shards_agree_mirror_norm(stv):
    if not _big_gpu((8 << 34) + (4 << 30)):
        pytest.skip("needs a 180 GB B200 (128 GiB state)")
    circ = C.config(4)
    n = circ.n
    rng = np.random.default_rng(4)
    y = np.unique(rng.integers(0, 1 << n, size=1 << 26, dtype=np.uint64))
    res = {}
    for g in (0, 1, 2):
        st = stv.State(n, "c64", virtual_g=g) if g else stv.State(n, "c64")
        st.set_basis(0)
        st.apply(circ.gates)
        res[g] = (st.amplitudes(y), st.norm(), st.stats())
        if g == 0:                          # mirror: C^dagger C |0> = |0>
            st.apply(C.inverse_gates(circ.gates))
            a0 = st.amplitudes(np.array([0, 1, (1 << n) - 1], dtype=np.uint64))
        st.close()
        del st
        _free()
    base = res[0][0]
    for g in (1, 2):
        d = float(np.max(np.abs(res[g][0] - base)))
        ov = np.vdot(base, res[g][0])
        fid = abs(ov) ** 2 / (np.vdot(base, base).real * np.vdot(res[g][0], res[g][0]).real)
        record(f"c4_c64_virtual_g{g}_vs_G1", n=n, sampled=int(y.size), max_abs=d, fidelity_sampled=fid,
               norm=res[g][1], remaps=res[g][2]["n_pass"]["remap"])
        assert d <= 2e-6 and fid >= 1 - 1e-5
        assert res[g][2]["n_pass"]["remap"] > 0
    record("c4_c64_mirror", n=n, amp0_sq=abs(a0[0]) ** 2, norm=res[0][1])
    assert abs(res[0][1] - 1) < 1e-4
    assert abs(a0[0]) ** 2 >= 1 - 1e-5 and abs(a0[1]) < 1e-4 and abs(a0[2]) < 1e-4


def test_c5_proxy_weak34_g3(stv):
    """c5 (n=37, 1 TiB over 8 GPUs with 3 global qubits) does not fit one B200.  Its proxy:
    the weak-ladder circuit at n=34 (same 6x6 grid family, gate set and seed as c5's ladder,
    inputs.circuits.weak_ladder) run with g=3 virtual shards -- the 8-shard partition c5 uses,
    every remap through the pack -> exchange -> unpack schedule -- against the unsharded run
    on 2^24 sampled amplitudes (2e-6, F >= 1 - 1e-5 over the sample)."""
    if not _big_gpu((8 << 34) + (4 << 30)):
        pytest.skip("needs a 180 GB B200 (128 GiB state)")
    circ = C.weak_ladder(34)
    n = circ.n
    rng = np.random.default_rng(5)
    y = np.unique(rng.integers(0, 1 << n, size=1 << 24, dtype=np.uint64))
    res = {}
    for g in (0, 3):
        st = stv.State(n, "c64", virtual_g=g) if g else stv.State(n, "c64")
        st.set_basis(0)
        st.apply(circ.gates)
        res[g] = (st.amplitudes(y), st.norm(), st.stats())
        st.close()
        del st
        _free()
    base, sh = res[0][0], res[3][0]
    d = float(np.max(np.abs(sh - base)))
    fid = abs(np.vdot(base, sh)) ** 2 / (np.vdot(base, base).real * np.vdot(sh, sh).real)
    record("c5_proxy_weak34_virtual_g3_vs_G1", n=n, sampled=int(y.size), max_abs=d, fidelity_sampled=fid,
           norm=res[3][1], remaps=res[3][2]["n_pass"]["remap"])
    assert d <= 2e-6 and fid >= 1 - 1e-5
    assert res[3][2]["n_pass"]["remap"] > 0
    assert abs(res[3][1] - 1) < 1e-4
