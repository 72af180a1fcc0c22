"""Pins of the CPU oracle against facts fixed by the paper and by mathematics
(-m "not gpu").  None of these re-types the oracle's formulas: each checks an
identity, a printed value, a closed form, or an independent (level-2 dense
Kronecker) evaluation, chosen so that a dropped term, a wrong sign/index or a
transposed operand in oracle/sv_oracle.c fails at least one of them.
"""
import cmath
import math

import numpy as np
import pytest

import oracle
from inputs import circuits as C

M = oracle.gate_matrix
I2 = np.eye(2)
X = np.array([[0, 1], [1, 0]], dtype=complex)
Y = np.array([[0, -1j], [1j, 0]])
Z = np.diag([1, -1]).astype(complex)
W_ = (X + Y) / math.sqrt(2)
SWAPM = np.eye(4)[[0, 2, 1, 3]]


def close(a, b, tol=1e-14):
    return np.max(np.abs(np.asarray(a) - np.asarray(b))) <= tol


# --------------------------------------------------------------------------
# gate-table pins (App. A)
# --------------------------------------------------------------------------
ALL_GATES = [("h", ()), ("x", ()), ("y", ()), ("z", ()), ("s", ()), ("t", ()),
             ("sx", ()), ("sy", ()), ("sw", ()), ("cz", ()), ("cnot", ()), ("swap", ()),
             ("cphase", ((1, 3),)), ("fsim", ((1, 2), (1, 6))), ("fsim", ((2, 7), (-3, 5)))]


@pytest.mark.parametrize("name,p", ALL_GATES)
def test_unitary(name, p):
    U = M(name, p)
    assert close(U.conj().T @ U, np.eye(U.shape[0]), 1e-15)
    assert close(M(name + "_dg", p), U.conj().T, 0)


def test_pauli_and_clifford_pins():
    H = M("h")
    assert close(H @ H, I2)
    assert close(H @ X @ H, Z)                      # H maps X <-> Z
    assert close(M("x"), X, 0) and close(M("y"), Y, 0) and close(M("z"), Z, 0)
    assert close(M("s") @ M("s"), Z)                # P = Z^{1/2}


def test_sqrt_x_pins():
    SX = M("sx")
    assert close(SX @ SX, X)                        # X^{1/2} squared
    assert close(SX, M("h") @ M("s") @ M("h"))      # X^{1/2} = H P H


def test_sqrt_y_pins():
    SY = M("sy")
    assert close(SY @ SY, -Y)                       # Y^{1/2}^2 = -Y (reading A3)
    # Eq. 2 / PAPER.md L647-653: Y^{1/2} H is diagonal (= e^{i pi/4} Z)
    assert close(SY @ M("h"), cmath.exp(1j * math.pi / 4) * Z)


def test_sqrt_w_pins():
    SW = M("sw")
    T = M("t")
    assert close(SW, T @ M("sx") @ T.conj().T)      # reading A4
    assert close(SW @ SW, W_)                       # W = (X+Y)/sqrt 2


def test_t_family_pins():
    T = M("t")
    assert close(np.linalg.matrix_power(T, 8), I2)  # T^8 = I
    assert close(T @ T, M("s"))                     # P = T^2
    assert close(np.linalg.matrix_power(T, 4), Z)   # Z = T^4
    assert close(T, np.diag([1, cmath.exp(1j * math.pi / 4)]))


@pytest.mark.parametrize("phi", [(1, 6), (-3, 7), (0, 1)])
def test_fsim_half_pi_is_swap_times_diag(phi):
    # reading A5: fSim(pi/2, phi) = SWAP . diag(1, -i, -i, e^{-i phi})
    ph = phi[0] * math.pi / phi[1]
    D = np.diag([1, -1j, -1j, cmath.exp(-1j * ph)])
    assert close(M("fsim", ((1, 2), phi)), SWAPM @ D)
    assert close(M("fsim", ((1, 2), phi)), D @ SWAPM)
    # fSim(0, phi) = CPHASE(-phi)
    assert close(M("fsim", ((0, 1), phi)), M("cphase", ((-phi[0], phi[1]),)))


def test_cphase_rk():
    for k in range(1, 8):
        U = M("cphase", ((2, 1 << k),))
        assert close(U, np.diag([1, 1, 1, cmath.exp(2j * math.pi / 2 ** k)]))
    assert close(M("cphase", ((1, 1),)), M("cz"))   # R_1 = CZ


def test_eq1_cnot_h_cz():
    # Eq. 1: (I x H) CNOT (I x H) = CZ; qubit 1 = MSB of
    # the 2-qubit index (reading A2), so "I x H" is H on qubit 0.
    U = oracle.kron_unitary(2, [("h", (0,), ()), ("cnot", (1, 0), ()), ("h", (0,), ())])
    assert close(U, M("cz"))
    # footnote: CNOT = (I x H) CZ (I x H)
    U = oracle.kron_unitary(2, [("h", (0,), ()), ("cz", (1, 0), ()), ("h", (0,), ())])
    assert close(U, M("cnot"))


def test_paper_printed_kronecker_products(golden):
    g = golden["paper_kron_products"]
    cx = lambda m: np.array([[complex(*e) for e in row] for row in m])
    Hp = M("h") * math.sqrt(2)
    Xp = M("sx") * 2
    Yp = M("sy") * 2
    assert close(np.kron(Hp, Hp), g["HpHp_scale"] * cx(g["HpHp"]), 1e-14)
    assert close(np.kron(Xp, Xp), g["XpXp_scale"] * cx(g["XpXp"]), 1e-14)
    lead = complex(*g["YpYp_leading_factor"])
    assert close(np.kron(Yp, Yp), g["YpYp_scale"] * lead * cx(g["YpYp"]), 1e-14)


def test_cnot_orientation():
    # CNOT(c=1, t=0) on |10> (index 2) -> |11> (index 3); first-listed = control
    psi = np.zeros(4, complex)
    psi[2] = 1
    oracle.apply(2, psi, [("cnot", (1, 0), ())])
    assert psi[3] == 1 and abs(psi).sum() == 1
    psi = np.zeros(4, complex)
    psi[1] = 1                                      # |01>: control (qubit 1) = 0
    oracle.apply(2, psi, [("cnot", (1, 0), ())])
    assert psi[1] == 1


# --------------------------------------------------------------------------
# index iteration: level 1 vs the dense Kronecker brute force
# --------------------------------------------------------------------------
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("seed", [1, 2])
def test_level1_matches_kronecker(n, seed):
    circ = C.random_circuit(n, 40, seed)
    U = oracle.kron_unitary(n, circ.gates)
    e = np.zeros(1 << n, complex)
    e[circ.x0] = 1
    ref = U @ e
    psi = oracle.run(circ)
    assert close(psi, ref, 1e-12)
    # whole-operator check on a random dense input (not just a basis vector)
    rng = np.random.default_rng(seed)
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    w = v.copy()
    oracle.apply(n, w, circ.gates)
    assert close(w, U @ v, 1e-11)


def test_kronecker_padding_is_definition():
    # level-2 padding pinned by np.kron on adjacent qubits: gate on qubits
    # (2,1) of 3 = I (x) U with qubit 2 as MSB
    U = M("u2", C.random_unitary(4, C.SplitMix64(5)))
    P = oracle.padded(3, "u2", (2, 1), C.random_unitary(4, C.SplitMix64(5)))
    assert close(P, np.kron(U, I2), 1e-15)
    P = oracle.padded(3, "h", (0,))
    assert close(P, np.kron(np.eye(4), M("h")), 0)


# --------------------------------------------------------------------------
# whole-circuit closed forms (PAPER.md L640 footnote, L1058-1060; textbook)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("n", [1, 4, 11])
def test_hadamard_layer_uniform(n):
    circ = C.Circuit("hn", n, [("h", (q,), ()) for q in range(n)])
    psi = oracle.run(circ)
    assert close(psi, np.full(1 << n, 2 ** (-n / 2)), 1e-15)


@pytest.mark.parametrize("n", [2, 5, 12])
def test_ghz(n):
    gates = [("h", (n - 1,), ())] + [("cnot", (q, q - 1), ()) for q in range(n - 1, 0, -1)]
    psi = oracle.run(C.Circuit("ghz", n, gates))
    ref = np.zeros(1 << n, complex)
    ref[0] = ref[-1] = 1 / math.sqrt(2)
    assert close(psi, ref, 1e-15)


@pytest.mark.parametrize("n", [3, 5, 7, 10])
def test_qft_closed_form(n):
    # reading A7: psi[y] = 2^{-n/2} exp(2 pi i x y / 2^n)
    circ = C.qft_circuit(n, tail=0, seed=3)
    psi = oracle.run(circ)
    y = np.arange(1 << n)
    ref = 2 ** (-n / 2) * np.exp(2j * np.pi * ((circ.x0 * y) % (1 << n)) / (1 << n))
    assert close(psi, ref, 1e-12)


def test_c3_tail_keeps_phase_state():
    # after the QFT, CNOT/X are permutations and CZ/T are phases: |psi_y| stays 2^{-n/2}
    circ = C.qft_circuit(12, tail=200, seed=3)
    psi = oracle.run(circ)
    assert close(np.abs(psi), np.full(1 << 12, 2 ** -6), 1e-13)


def test_norm_and_mirror():
    circ = C.config(1)
    psi = oracle.run(circ, nthreads=4)
    assert abs(oracle.norm(psi) - 1) < 1e-13
    back = oracle.apply(circ.n, psi.copy(), C.inverse_gates(circ.gates))
    e = np.zeros(1 << circ.n, complex)
    e[0] = 1
    assert close(back, e, 1e-12)
    r = C.random_circuit(9, 120, 4)
    psi = oracle.run(r)
    back = oracle.apply(9, psi, C.inverse_gates(r.gates))
    e = np.zeros(1 << 9, complex)
    e[r.x0] = 1
    assert close(back, e, 1e-12)


def test_threads_bitwise_identical():
    circ = C.random_circuit(14, 60, 9)
    a = oracle.run(circ, nthreads=1)
    b = oracle.run(circ, nthreads=8)
    assert np.array_equal(a, b)


def test_compare_metrics():
    a = np.zeros(8, complex)
    a[0] = 1
    b = a * 1j
    r = oracle.compare(b, a)
    assert r["fidelity"] == pytest.approx(1.0) and r["max_abs"] == pytest.approx(math.sqrt(2))


# --------------------------------------------------------------------------
# the paper's bitmask examples (Sec. 4.3) -- pins of readings A1 and of the
# diagonal-phase rules the CUDA path's diag encoding is later tested against
# --------------------------------------------------------------------------
def _bits(s):
    return int(s, 2)


def test_cz_complete_graph_masks(golden):
    g = golden["paper_bitmasks"]["cz_complete_graph_4q"]
    masks = [_bits(s) for s in g["masks"]]
    # m_k = partners of qubit k (LSB convention)
    for k in range(4):
        assert masks[k] == sum(1 << l for l in range(4) if l != k)
    assert sum(bin(m).count("1") for m in masks) == g["total_set_bits"]
    # sign rule: (sum_{k in j} popc(m_k & j)) & 2
    # equals the brute-force parity of CZ pairs with both bits set
    for j in range(16):
        cnt = sum(bin(masks[k] & j).count("1") for k in range(4) if j >> k & 1)
        pairs = sum(1 for a in range(4) for b in range(a + 1, 4) if j >> a & 1 and j >> b & 1)
        assert bool(cnt & 2) == bool(pairs & 1)
    # the same signs from the oracle applying the six CZ gates one by one
    gates = [("cz", (a, b), ()) for a in range(4) for b in range(a + 1, 4)]
    for j in range(16):
        psi = oracle.run(C.Circuit("cz", 4, gates), x0=j)
        cnt = sum(bin(masks[k] & j).count("1") for k in range(4) if j >> k & 1)
        assert psi[j] == (-1 if cnt & 2 else 1)


def test_fig_cz_and_reorder_masks(golden):
    g = golden["paper_bitmasks"]
    f = g["fig_CZ"]
    masks = [0] * f["n"]
    for a, b in f["cz"]:
        masks[a] |= 1 << b
        masks[b] |= 1 << a
    assert [format(m, "03b") for m in masks] == f["masks"]
    r = g["fig_reorder"]
    assert format(sum(1 << q for q in r["t_qubits"]), "04b") == r["t_mask"]
    assert format(sum(1 << q for q in r["sx_qubits"]), "04b") == r["sx_mask"]
    assert format(sum(1 << q for q in r["sy_qubits"]), "04b") == r["sy_mask"]
    one = {}
    for a, b in r["cz"]:
        one[str(max(a, b))] = format(1 << min(a, b), "04b")
    assert one == r["cz_onesided_masks"]


def test_gray_code(golden):
    seq = golden["paper_bitmasks"]["gray3"]["sequence"]
    assert [k ^ (k >> 1) for k in range(8)] == seq
    assert all(bin(seq[i] ^ seq[(i + 1) % 8]).count("1") == 1 for i in range(8))


def test_t_octant_rule():
    # T-layer phase = exp(i pi/4)^{popcount(m & j) mod 8}
    m = 0b1011
    gates = [("t", (q,), ()) for q in range(4) if m >> q & 1] * 3
    for j in range(16):
        psi = oracle.run(C.Circuit("t", 4, gates), x0=j)
        k = (3 * bin(m & j).count("1")) % 8
        assert abs(psi[j] - cmath.exp(1j * math.pi / 4 * k)) < 1e-15


# --------------------------------------------------------------------------
# generators: determinism and structure (inputs/, shared by both sides)
# --------------------------------------------------------------------------
def test_config_shapes_and_hashes():
    expect = {1: (16, 380, 60), 2: (30, 723, 123), 3: (32, 744, None), 4: (34, 576, 100), 5: (37, 625, 107)}
    for c, (n, g, g2) in expect.items():
        circ = C.config(c)
        assert circ.n == n and len(circ.gates) == g
        if g2 is not None:
            assert sum(len(x[1]) == 2 for x in circ.gates) == g2
        assert C.config(c).sha256() == circ.sha256()
        assert C.from_text(circ.text()).gates == circ.gates


def test_coupler_patterns_cover_grid():
    for (R, Cc, rm) in [(4, 4, 0), (5, 6, 0), (6, 6, 2), (6, 7, 5)]:
        pats = C.coupler_patterns(R, Cc, rm)
        allp = [p for pat in pats for p in pat]
        assert len(allp) == len(set(allp))
        for pat in pats:                              # each class is a matching
            qs = [q for p in pat for q in p]
            assert len(qs) == len(set(qs))
    assert sum(len(p) for p in C.coupler_patterns(4, 4)) == 24
    assert sum(len(p) for p in C.coupler_patterns(5, 6)) == 49


# ------------------ single-amplitude paths (sampled full-size parity) ------------------
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_monomial_amplitudes_vs_run(seed):
    # brute force: the full gate-by-gate state of a random permutation/phase circuit
    # applied to a random (non-basis) input state
    n = 10
    circ = C.random_circuit(n, 300, seed, kinds=["x", "cnot", "swap", "z", "s", "t", "cz", "cphase"])
    rng = np.random.default_rng(seed)
    psi0 = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    psi0 /= np.linalg.norm(psi0)
    full = oracle.apply(n, psi0.copy(), circ.gates)
    ys = np.arange(1 << n, dtype=np.uint64)
    got = oracle.monomial_amplitudes(n, circ.gates, lambda x: psi0[x.astype(np.int64)], ys)
    assert close(got, full, 1e-13)


def test_monomial_amplitudes_rejects_dense_gates():
    with pytest.raises(ValueError):
        oracle.monomial_amplitudes(2, [("h", (0,), ())], lambda x: np.ones(x.size), [0])


@pytest.mark.parametrize("n", [8, 14])
def test_c3_paths_vs_run(n):
    # c3 shape: QFT closed form followed by the CNOT/X/CZ/T tail, against run()
    circ = C.qft_circuit(n, tail=200, seed=3)
    nq = len(C.qft_gates(n))
    psi = oracle.run(circ)
    ys = np.arange(1 << n, dtype=np.uint64)
    got = oracle.monomial_amplitudes(n, circ.gates[nq:], lambda x: oracle.qft_basis_amplitudes(n, circ.x0, x), ys)
    assert close(got, psi, 1e-12)


@pytest.mark.parametrize("n", [3, 5, 7, 10])
def test_qft_basis_amplitudes_vs_run(n):
    circ = C.qft_circuit(n, tail=0, seed=5)
    psi = oracle.run(circ)
    got = oracle.qft_basis_amplitudes(n, circ.x0, np.arange(1 << n))
    assert close(got, psi, 1e-12)


# --------------------------------------------------------------------------
# complex64-storage mode (reading A19: the full-state c4 oracle, 128 GiB)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("n", [3, 10])
def test_c64store_closed_forms(n):
    """H^n|0> is uniform and the QFT of a basis state is 2^{-n/2} e^{2 pi i x y / 2^n} (A7),
    to complex64 rounding (each gate rounded once when stored)."""
    h = oracle.run_c64store(C.Circuit("hn", n, [("h", (q,), ()) for q in range(n)]))
    assert h.dtype == np.complex64
    assert close(h, np.full(1 << n, 2 ** (-n / 2)), 1e-7)
    circ = C.qft_circuit(n, tail=0, seed=3)
    y = np.arange(1 << n)
    ref = 2 ** (-n / 2) * np.exp(2j * np.pi * ((circ.x0 * y) % (1 << n)) / (1 << n))
    assert close(oracle.run_c64store(circ), ref, 1e-6)


@pytest.mark.parametrize("n,seed", [(9, 1), (12, 2)])
def test_c64store_vs_run_and_grid(n, seed):
    """Random circuits of every gate kind and the c4-shaped grid circuit at small size: the
    complex64-storage run stays within complex64 rounding of the complex128 oracle
    (per-gate rounding ~2^-24 relative, random-walk accumulated) and keeps the norm."""
    for circ in (C.random_circuit(n, 300, seed), C.grid_circuit("g", 3, 4, 0, 14, "fsim", seed)):
        a = oracle.run_c64store(circ)
        b = oracle.run(circ)
        assert np.max(np.abs(a.astype(np.complex128) - b)) < 2e-6
        assert abs(np.vdot(a, a).real - 1) < 1e-5
