"""Measurement sampling.

CPU (-m "not gpu"): the oracle sampler pinned to the published splitmix64 outputs,
to basis states and to the Born rule (chi-square).
GPU (-m gpu): sv_sample through the C ABI against the ORACLE's own state
(oracle.run): every sample must bracket the oracle's logical-order CDF within the
bound implied by the per-amplitude bar, and agree index for index with the oracle
sampler except within rounding of a CDF boundary; plus basis states, virtual
shards and a Born-rule chi-square.  No GPU-produced value (amplitudes, frame) is
passed to any oracle call.
"""
import numpy as np
import pytest

import oracle
from inputs import circuits as C


# --------------------------- CPU: the oracle sampler ---------------------------
def test_splitmix64_reference_outputs():
    # Vigna's splitmix64: state 0 -> 0xe220a8397b1dcdaf, 0x6e789e6aa1b965f4 and the
    # widely used seed-1234567 test sequence
    assert [oracle.splitmix64(0, s) for s in range(2)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4]
    assert [oracle.splitmix64(1234567, s) for s in range(3)] == [
        6457827717110365317, 3203168211198807973, 9817491932198370423]


def test_uniforms_in_unit_interval_and_uniform():
    u = oracle.uniforms(7, 64000)
    assert u.min() >= 0 and u.max() < 1
    h = np.histogram(u, bins=64, range=(0, 1))[0]
    chi2 = float(np.sum((h - 1000.0) ** 2 / 1000.0))
    assert chi2 < 120          # 63 dof: p ~ 1e-5


@pytest.mark.parametrize("x", [0, 5, 1023])
def test_sample_basis_state(x):
    psi = np.zeros(1024, dtype=np.complex128)
    psi[x] = 1j
    assert np.all(oracle.sample(psi, 11, 100) == x)


def test_sample_born_rule_chi_square():
    rng = np.random.default_rng(3)
    psi = rng.normal(size=64) + 1j * rng.normal(size=64)
    p = np.abs(psi) ** 2 / np.sum(np.abs(psi) ** 2)
    shots = 200000
    s = oracle.sample(psi, 5, shots)
    h = np.bincount(s.astype(np.int64), minlength=64)
    chi2 = float(np.sum((h - shots * p) ** 2 / (shots * p)))
    assert chi2 < 120          # 63 dof


def test_sample_two_outcomes_half_half():
    psi = np.zeros(4, dtype=np.complex128)
    psi[0] = 1 / np.sqrt(2)
    psi[3] = 1j / np.sqrt(2)
    s = oracle.sample(psi, 1, 100000)
    assert set(np.unique(s)) == {0, 3}
    assert abs(np.mean(s == 0) - 0.5) < 0.01


# --------------------------- GPU: sv_sample ---------------------------
@pytest.fixture(scope="module")
def stv():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2008_00216_b200 as m
    m.lib()
    return m


def _bracket_check(got, ref, seed, eps):
    """Every GPU sample j must satisfy cdf(j-1) - eps <= u * total <= cdf(j) + eps for the
    ORACLE's state (oracle.run), with u the oracle's own counter-based uniforms: the
    definition in include/sv.h, evaluated on independent amplitudes."""
    p = np.abs(ref) ** 2
    cdf = np.cumsum(p)
    total = cdf[-1]
    t = oracle.uniforms(seed, got.size) * total
    j = got.astype(np.int64)
    assert np.all((j >= 0) & (j < ref.size))
    lo = np.where(j > 0, cdf[np.maximum(j - 1, 0)], 0.0)
    hi = cdf[j]
    bad = np.nonzero((t < lo - eps) | (t > hi + eps) | (p[j] == 0))[0]
    assert bad.size == 0, (bad[:5], t[bad[:5]], lo[bad[:5]], hi[bad[:5]])


def _eps(ref, bar):
    # per-amplitude bar |d| <= bar  =>  | |a+d|^2 - |a|^2 | <= 2 |a| bar + bar^2: summed over
    # all indices it bounds the CDF shift; doubled for the u * total term
    return 2.0 * (2.0 * bar * float(np.sum(np.abs(ref))) + ref.size * bar * bar) + 1e-15


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n,seed", [(5, 1), (12, 2), (16, 3)])
def test_gpu_sample_matches_oracle_cdf(stv, n, seed, dtype):
    circ = C.random_circuit(n, 12 * n, seed)
    ref = oracle.run(circ)
    st = stv.State(n, dtype)
    st.set_basis(circ.x0)
    st.apply(circ.gates)
    shots = 20000
    got = st.sample(shots, seed=seed + 100)
    st.close()
    _bracket_check(got, ref, seed + 100, _eps(ref, 2e-6 if dtype == "c64" else 1e-12))
    want = oracle.sample(ref, seed + 100, shots)
    same = int(np.count_nonzero(got == want))
    # only draws within rounding of a CDF boundary may differ
    assert same >= shots - (1 if dtype == "c128" else shots // 100), same


@pytest.mark.gpu
def test_gpu_sample_born_rule_vs_oracle_state(stv):
    circ = C.random_circuit(10, 150, 9)
    ref = oracle.run(circ)
    p = np.abs(ref) ** 2
    st = stv.State(10, "c64")
    st.set_basis(circ.x0)
    st.apply(circ.gates)
    shots = 400000
    s = st.sample(shots, seed=4)
    st.close()
    h = np.bincount(s.astype(np.int64), minlength=1024)
    m = p * shots > 20
    chi2 = float(np.sum((h[m] - shots * p[m]) ** 2 / (shots * p[m])))
    assert chi2 < int(m.sum()) + 6 * np.sqrt(2 * int(m.sum()))


@pytest.mark.gpu
@pytest.mark.parametrize("x", [0, 12345, (1 << 20) - 1])
def test_gpu_sample_basis(stv, x):
    st = stv.State(20, "c64")
    st.set_basis(x)
    assert np.all(st.sample(1000, seed=x) == x)
    st.apply([("x", (3,), ()), ("swap", (0, 19), ())])   # relabel only: frame changes, data does not
    y = x ^ (1 << 3)
    y = (y & ~((1 << 0) | (1 << 19))) | (((y >> 19) & 1) << 0) | (((y >> 0) & 1) << 19)
    assert np.all(st.sample(1000, seed=1) == y)
    st.close()


@pytest.mark.gpu
@pytest.mark.parametrize("g", [1, 2, 3])
def test_gpu_sample_virtual_shards(stv, g):
    circ = C.random_circuit(14, 150, 5)
    ref = oracle.run(circ)
    st = stv.State(14, "c64", virtual_g=g)
    st.set_basis(circ.x0)
    st.apply(circ.gates)
    got = st.sample(5000, seed=8)
    st.close()
    _bracket_check(got, ref, 8, _eps(ref, 2e-6))


@pytest.mark.gpu
def test_gpu_sample_errors_and_empty(stv):
    st = stv.State(6, "c64")
    assert st.sample(0).size == 0
    st.close()
