"""GPU parity: the CUDA path through the C ABI vs the CPU oracle (-m gpu).

Bars (BASELINE.json north_star): complex64 per-amplitude |delta| <= 2e-6 and
fidelity >= 1 - 1e-5; complex128 |delta| <= 1e-12.  Inputs are the seeded
generators of inputs/ (no value ever comes from the CUDA path).
"""
import math

import numpy as np
import pytest

import oracle
from inputs import circuits as C

pytestmark = pytest.mark.gpu

TOL = {"c64": 2e-6, "c128": 1e-12}


@pytest.fixture(scope="module")
def stv():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2008_00216_b200 as m
    m.lib()
    return m


def run_gpu(stv, circ, dtype="c64", **kw):
    st = stv.State(circ.n, dtype)
    st.set_basis(circ.x0)
    st.apply(circ.gates, **kw)
    psi = st.amplitudes()
    stats = st.stats()
    st.close()
    return psi, stats


def assert_parity(psi, ref, dtype):
    r = oracle.compare(psi, ref)
    assert r["max_abs"] <= TOL[dtype], r
    if dtype == "c64":
        assert r["fidelity"] >= 1 - 1e-5, r
    return r


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,seed", [(1, 1), (2, 2), (4, 3), (6, 4), (9, 5), (12, 6), (15, 7), (18, 8)])
def test_random_circuits_all_kinds(stv, n, seed, dtype):
    circ = C.random_circuit(n, 150, seed)
    psi, _ = run_gpu(stv, circ, dtype)
    assert_parity(psi, oracle.run(circ), dtype)


@pytest.mark.parametrize("kw", [dict(kmax=1), dict(kmax=2), dict(kmax=3), dict(kmax=4),
                                dict(tile_bits=8, low_bits=3), dict(tile_bits=13, low_bits=5),
                                dict(tile_bits=10, low_bits=0), dict(budget=400), dict(budget=20),
                                dict(flags=2), dict(flags=4), dict(flags=8), dict(flags=16),
                                dict(flags=32), dict(flags=128), dict(flags=32 | 128),
                                dict(flags=0x400), dict(flags=0x800)])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_planner_options(stv, kw, dtype):
    circ = C.random_circuit(17, 300, 42)
    psi, _ = run_gpu(stv, circ, dtype, **kw)
    assert_parity(psi, oracle.run(circ), dtype)


@pytest.mark.parametrize("n,seed", [(20, 9), (21, 12), (22, 10)])
def test_random_circuits_all_kinds_tc(stv, n, seed):
    """Random circuits of every gate kind at n >= 20, where complex64 passes have full 12-bit
    tiles and run on the tensor-core kernel (smaller states run on the CUDA-core pass)."""
    circ = C.random_circuit(n, 250, seed)
    psi, st = run_gpu(stv, circ, "c64")
    assert st["n_tc_pass"] > 0
    assert_parity(psi, oracle.run(circ), "c64")


@pytest.mark.parametrize("kw", [dict(kmax=1), dict(kmax=2), dict(kmax=3), dict(low_bits=5), dict(low_bits=7),
                                dict(budget=400), dict(flags=2), dict(flags=4), dict(flags=16),
                                dict(flags=128), dict(flags=0x400), dict(flags=0x800)])
def test_planner_options_tc(stv, kw):
    """The planner options on the tensor-core path (n = 20: full 12-bit tiles, complex64)."""
    circ = C.random_circuit(20, 300, 43)
    psi, st = run_gpu(stv, circ, "c64", **kw)
    assert st["n_tc_pass"] > 0
    assert_parity(psi, oracle.run(circ), "c64")


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_c1_config(stv, dtype):
    circ = C.config(1)
    psi, st = run_gpu(stv, circ, dtype)
    assert_parity(psi, oracle.run(circ), dtype)
    assert st["n_kernels"] >= 1


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_qft_closed_form(stv, dtype):
    n = 20
    circ = C.qft_circuit(n, tail=0, seed=3)
    psi, _ = run_gpu(stv, circ, dtype)
    y = np.arange(1 << n)
    ref = 2 ** (-n / 2) * np.exp(2j * np.pi * ((circ.x0 * y) % (1 << n)) / (1 << n))
    assert np.max(np.abs(psi - ref)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_c3_reduced(stv, dtype):
    circ = C.qft_circuit(22, tail=200, seed=3)
    psi, _ = run_gpu(stv, circ, dtype)
    assert_parity(psi, oracle.run(circ), dtype)
    # phase state: |psi_y| = 2^{-n/2} for all y (permutations + phases after the QFT)
    assert np.max(np.abs(np.abs(psi) - 2 ** -11)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_grid_fsim_reduced(stv, dtype):
    circ = C.grid_circuit("g", 4, 5, 0, 20, "fsim", 2)
    psi, _ = run_gpu(stv, circ, dtype)
    assert_parity(psi, oracle.run(circ), dtype)


@pytest.mark.parametrize("g", [1, 2, 3])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_virtual_shards(stv, g, dtype):
    circ = C.random_circuit(16, 250, 60 + g)
    st = stv.State(circ.n, dtype, virtual_g=g)
    st.set_basis(circ.x0)
    st.apply(circ.gates, tile_bits=8, low_bits=3)
    s = st.stats()
    psi = st.amplitudes()
    st.close()
    assert s["n_pass"]["remap"] > 0
    assert_parity(psi, oracle.run(circ), dtype)


@pytest.mark.parametrize("g", [1, 2, 3])
def test_virtual_shards_n24_pack_exchange(stv, g):
    """Virtual shards run every pass per shard with that rank's encoding and every remap
    through the distributed pack -> exchange -> unpack path (device copies in place of
    ncclSend/ncclRecv), default planner options, n = 24."""
    circ = C.grid_circuit("g24", 4, 6, 0, 10, "fsim", 20 + g)
    st = stv.State(circ.n, "c64", virtual_g=g)
    st.set_basis(circ.x0)
    st.apply(circ.gates)
    s = st.stats()
    psi = st.amplitudes()
    st.close()
    assert s["n_pass"]["remap"] > 0 and s["remap_bytes"] > 0
    assert_parity(psi, oracle.run(circ), "c64")


def test_virtual_shards_grid(stv):
    circ = C.grid_circuit("g", 4, 5, 0, 12, "fsim", 9)
    st = stv.State(circ.n, "c64", virtual_g=3)
    st.apply(circ.gates)
    psi = st.amplitudes()
    st.close()
    assert_parity(psi, oracle.run(circ), "c64")


def test_incremental_apply_keeps_frame(stv):
    circ = C.random_circuit(14, 200, 77)
    st = stv.State(14)
    st.set_basis(circ.x0)
    for k in range(0, 200, 37):
        st.apply(circ.gates[k:k + 37])
    perm, xm = st.frame()
    psi = st.amplitudes()
    st.close()
    assert_parity(psi, oracle.run(circ), "c64")
    assert sorted(perm) == list(range(14))


def test_norm_deterministic(stv):
    circ = C.random_circuit(20, 200, 3)
    st = stv.State(20)
    st.apply(circ.gates)
    a = st.norm()
    b = st.norm()
    st.close()
    assert a == b and abs(a - 1) < 1e-5


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n", [1, 7, 13, 22])
def test_norm_vs_host_fp64_sum(stv, n, dtype):
    """sv_norm of a NON-normalised buffer (seeded normal values written into the wrapped
    tensor) against the fp64 host sum of |a|^2, 1e-12 relative."""
    import torch
    rng = np.random.default_rng(n)
    real = np.float32 if dtype == "c64" else np.float64
    host = (rng.normal(size=2 << n) * 3.0).astype(real)
    st = stv.State(n, dtype)
    st.tensor.copy_(torch.from_numpy(host).to(st.tensor.device))
    torch.cuda.synchronize()
    got = st.norm()
    st.close()
    want = float(np.sum(host.astype(np.float64) ** 2))
    assert abs(got - want) <= 1e-12 * want, (got, want)


def test_uniform_init_and_get_amplitudes(stv):
    st = stv.State(12, "c128")
    st.set_uniform()
    idx = np.array([0, 5, 4095, 17], dtype=np.uint64)
    v = st.amplitudes(idx)
    assert np.allclose(v, 2 ** -6, atol=1e-15)
    assert abs(st.norm() - 1) < 1e-13
    with pytest.raises(stv.SvError):
        st.amplitudes(np.array([1 << 12], dtype=np.uint64))
    st.close()


def test_invalid_gate_launches_nothing(stv):
    st = stv.State(6)
    st.set_basis(3)
    with pytest.raises(stv.SvError, match="gate 1"):
        st.apply([("h", (0,), ()), ("cz", (2, 9), ())])
    psi = st.amplitudes()
    st.close()
    e = np.zeros(64)
    e[3] = 1
    assert np.array_equal(psi, e)


def test_empty_and_relabel_only(stv):
    st = stv.State(10)
    st.set_basis(5)
    st.apply([])
    st.apply([("x", (0,), ()), ("swap", (0, 9), ()), ("x", (3,), ())])
    psi = st.amplitudes()
    st.close()
    ref = oracle.run(C.Circuit("r", 10, [("x", (0,), ()), ("swap", (0, 9), ()), ("x", (3,), ())], x0=5))
    assert np.array_equal(psi, ref)


def test_read_state_raw(stv):
    circ = C.random_circuit(13, 100, 8)
    st = stv.State(13)
    st.set_basis(circ.x0)
    st.apply(circ.gates)
    raw = st.read_state()
    wide = st.amplitudes()
    st.close()
    assert raw.dtype == np.complex64 and np.array_equal(raw.astype(np.complex128), wide)


def test_bitwise_reproducible(stv):
    circ = C.config(1)
    a, _ = run_gpu(stv, circ)
    b, _ = run_gpu(stv, circ)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("budget", [20, 100, 450, 2000])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_grid_fsim_budgets(stv, budget, dtype):
    circ = C.grid_circuit("g", 4, 5, 0, 20, "fsim", 2)
    psi, _ = run_gpu(stv, circ, dtype, budget=budget)
    assert_parity(psi, oracle.run(circ), dtype)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_c2_shape_reduced(stv, dtype):
    # the c2 generator on a 4x6 grid (24 qubits), default options
    circ = C.grid_circuit("c2s", 4, 6, 0, 20, "fsim", 2)
    psi, _ = run_gpu(stv, circ, dtype)
    assert_parity(psi, oracle.run(circ, nthreads=16), dtype)


def test_plan_cache_hit_identical_and_frame_keyed(stv):
    """An identical call (same gates, frame, options) reuses the plan and its resident device
    blob (no planning, no upload) and gives bit-identical results; a different frame (after a
    relabel-only X) is a different key and still matches the oracle."""
    circ = C.config(1)
    st = stv.State(circ.n)
    st.set_basis(circ.x0)
    st.apply(circ.gates)
    a = st.amplitudes()
    cold = st.stats()
    st.set_basis(circ.x0)
    st.apply(circ.gates)
    b = st.amplitudes()
    warm = st.stats()
    assert np.array_equal(a, b)
    assert warm["h2d_bytes"] == 0 and cold["h2d_bytes"] > 0
    st.set_basis(circ.x0)
    st.apply([("x", (3,), ())] + list(circ.gates[:50]))      # X relabels the frame first
    st.apply(circ.gates[50:])
    c = st.amplitudes()
    st.set_basis(circ.x0)
    st.apply(circ.gates, flags=stv.OPT_NO_PLAN_CACHE)
    d = st.amplitudes()
    st.close()
    ref = oracle.run(C.Circuit("x+c1", circ.n, [("x", (3,), ())] + list(circ.gates), x0=circ.x0))
    assert_parity(c, ref, "c64")
    assert np.array_equal(a, d)


@pytest.mark.parametrize("dims", [(4, 5, 20, 2), (4, 6, 20, 3)])
def test_tc_block_variants_parity(stv, dims):
    """Tensor-core passes with per-block operator variants (a one-V-bit table or V-bit-controlled
    CNOT folded into two operators, one per 128-row TMEM block) and with the fully tile-uniform
    operators, against the oracle; the same circuit on the CUDA-core kernel agrees too."""
    from tests import blob_emu as BE
    R, Cc, cyc, seed = dims
    circ = C.grid_circuit("g", R, Cc, 0, cyc, "fsim", seed)
    blob, offs = stv.plan_blob(circ.n, circ.gates)
    nb = 0
    for po in offs:
        P = BE._at(blob, BE.Pass, po)
        if P.kind == 1 and P.grouped and P.ntc:
            nb += sum(1 for i in range(P.ntc) if BE._at(blob, BE.TcStep, po + P.tc_off + 32 * i).bvar)
    assert nb > 0
    ref = oracle.run(circ)
    psi, st = run_gpu(stv, circ, "c64")
    assert st["n_tc_pass"] > 0
    assert_parity(psi, ref, "c64")
    psi2, _ = run_gpu(stv, circ, "c64", flags=stv.OPT_NO_TC)
    assert_parity(psi2, ref, "c64")


@pytest.mark.parametrize("cfg", [1, 2])
def test_tma_staged_tc_pass_parity(stv, cfg):
    """Tensor-core passes staged with TMA tensor copies (SV_OPT_TMA: 5-D tensor map with an
    overlapping tile-base dim, SWIZZLE_128B tile layout, looped boxes) against the oracle."""
    circ = C.grid_circuit("g", 4, 5, 0, 12, "fsim", 20) if cfg == 1 else C.grid_circuit("g", 4, 6, 0, 12, "fsim", 21)
    ref = oracle.run(circ)
    a, st = run_gpu(stv, circ, "c64", flags=stv.OPT_TMA)
    assert st["n_tc_pass"] > 0
    assert_parity(a, ref, "c64")


_FUZZ_OPTS = [dict(), dict(kmax=1), dict(kmax=2), dict(kmax=3), dict(low_bits=5), dict(low_bits=6), dict(budget=400),
              dict(flags=2), dict(flags=16), dict(flags=128), dict(flags=0x400), dict(flags=0x800), dict(tile_bits=11),
              dict(tile_bits=13), dict(kmax=2, low_bits=5), dict(kmax=3, budget=400), dict(kmax=2, flags=0x800)]
_FUZZ_KINDS = [None, ["h", "cz", "t", "x", "cnot"], ["u1", "fsim"], ["u2", "cphase", "h"], ["cnot", "x", "cz", "t", "h"]]


@pytest.mark.parametrize("case", range(24))
def test_seeded_fuzz_full_tiles(stv, case):
    """Seeded draws of (circuit shape, planner options, dtype, virtual shards) at n = 20..22, where
    complex64 plans have full 12-bit tiles (tensor-core pass): the combinations the fixed option
    lists above do not enumerate (`tools/gpu_fuzz.py` is the long-running form of this test)."""
    rng = C.SplitMix64(77000 + case)
    n = 20 + rng.u(3)
    shape = rng.u(3)
    if shape == 0:
        circ = C.qft_circuit(n, 40 + rng.u(80), 500 + case, "fz")
    elif shape == 1 and n % 4 == 0:
        circ = C.grid_circuit("fz", 4, n // 4, 0, 6 + rng.u(6), "fsim" if rng.u(2) else "cz", 500 + case)
    else:
        circ = C.random_circuit(n, 150 + rng.u(250), 500 + case, _FUZZ_KINDS[rng.u(len(_FUZZ_KINDS))])
    kw = _FUZZ_OPTS[rng.u(len(_FUZZ_OPTS))]
    dtype = "c128" if rng.u(4) == 0 else "c64"
    g = (0, 0, 1, 2, 3)[rng.u(5)]
    st = stv.State(circ.n, dtype, virtual_g=g) if g else stv.State(circ.n, dtype)
    st.set_basis(circ.x0)
    st.apply(circ.gates, **kw)
    psi = st.amplitudes()
    st.close()
    assert_parity(psi, oracle.run(circ), dtype)
