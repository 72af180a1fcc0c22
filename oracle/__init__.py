"""oracle/ -- TEST INFRASTRUCTURE ONLY (see sv_oracle.c header).

Python face of the plain complex128 CPU oracle.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs
may import this package; the product package never does.

  run(circuit)           level 1: gate-by-gate in-place update (PAPER.md
                         L236-241), C + OpenMP, complex128
  kron_unitary(n, gates) level 2: every gate padded to a dense 2^n x 2^n
                         matrix and multiplied in order,
                         numpy, n <= 8 -- the "enormously wasteful" baseline
  gate_matrix(...)       the oracle's own gate table (sv_oracle.c)
  compare(psi, ref)      max |delta|, fidelity, norms
  monomial_amplitudes    single output amplitudes of permutation/phase circuits
                         (one row of each padded matrix), for sampled parity at
                         full size; qft_basis_amplitudes: the QFT closed form
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

KINDS = {"h": 0, "x": 1, "y": 2, "z": 3, "s": 4, "t": 5, "sx": 6, "sy": 7, "sw": 8,
         "cz": 9, "cnot": 10, "swap": 11, "cphase": 12, "fsim": 13, "u1": 14, "u2": 15}


class _Gate(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("adjoint", ctypes.c_int32),
                ("q0", ctypes.c_int32), ("q1", ctypes.c_int32),
                ("theta", ctypes.c_double), ("phi", ctypes.c_double),
                ("m", ctypes.POINTER(ctypes.c_double))]


def build(force: bool = False) -> str:
    """Compile sv_oracle.c (plain C, -O2, OpenMP) in-tree."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-fopenmp",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.oracle_gate_matrix.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                         ctypes.c_double, ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double)]
        L.oracle_run.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p,
                                 ctypes.POINTER(_Gate), ctypes.c_int64, ctypes.c_int]
        L.oracle_apply.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(_Gate),
                                   ctypes.c_int64, ctypes.c_int]
        L.oracle_run_c64store.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p,
                                          ctypes.POINTER(_Gate), ctypes.c_int64, ctypes.c_int]
        L.oracle_norm.argtypes = [ctypes.c_int, ctypes.c_void_p]
        L.oracle_norm.restype = ctypes.c_double
        _lib = L
    return _lib


def _angle(a):
    num, den = a
    return float(num) * np.pi / float(den)


def _split(name):
    if name.endswith("_dg"):
        return name[:-3], 1
    return name, 0


def _marshal(gates):
    arr = (_Gate * max(1, len(gates)))()
    keep = []
    for i, (name, qs, p) in enumerate(gates):
        base, adj = _split(name)
        g = arr[i]
        g.kind = KINDS[base]
        g.adjoint = adj
        g.q0 = qs[0]
        g.q1 = qs[1] if len(qs) > 1 else -1
        g.theta = g.phi = 0.0
        if base == "cphase":
            g.phi = _angle(p[0])
        elif base == "fsim":
            g.theta, g.phi = _angle(p[0]), _angle(p[1])
        if base in ("u1", "u2"):
            m = (ctypes.c_double * len(p))(*p)
            keep.append(m)
            g.m = m
        else:
            g.m = None
    return arr, keep


def gate_matrix(name: str, params: tuple = ()) -> np.ndarray:
    """The oracle's matrix for one gate (first-listed qubit = MSB)."""
    base, adj = _split(name)
    theta = phi = 0.0
    if base == "cphase":
        phi = _angle(params[0])
    elif base == "fsim":
        theta, phi = _angle(params[0]), _angle(params[1])
    m = (ctypes.c_double * 32)(*(params if base in ("u1", "u2") else ()))
    out = (ctypes.c_double * 32)()
    d = lib().oracle_gate_matrix(KINDS[base], adj, theta, phi, m, out)
    if d < 0:
        raise ValueError(name)
    a = np.array(out[: 2 * d * d]).reshape(d, d, 2)
    return a[..., 0] + 1j * a[..., 1]


def apply(n: int, psi: np.ndarray, gates, nthreads: int = 0) -> np.ndarray:
    """psi <- C psi in place (complex128, length 2^n)."""
    assert psi.dtype == np.complex128 and psi.size == 1 << n and psi.flags.c_contiguous
    arr, keep = _marshal(gates)
    rc = lib().oracle_apply(n, psi.ctypes.data, arr, len(gates), nthreads)
    if rc != 0:
        raise ValueError(f"oracle: bad gate {-rc - 1}")
    return psi


def run(circuit, nthreads: int = 0, gates=None, x0=None) -> np.ndarray:
    """Level 1: psi = U_G ... U_1 e_{x0} (complex128)."""
    n = circuit.n
    x0 = circuit.x0 if x0 is None else x0
    gates = circuit.gates if gates is None else gates
    psi = np.empty(1 << n, dtype=np.complex128)
    arr, keep = _marshal(gates)
    rc = lib().oracle_run(n, x0, psi.ctypes.data, arr, len(gates), nthreads)
    if rc != 0:
        raise ValueError(f"oracle: rc={rc}")
    return psi


def run_c64store(circuit, nthreads: int = 0) -> np.ndarray:
    """Level 1 with complex64 storage (reading A19): psi = U_G ... U_1 e_{x0}, each
    gate computed in complex128 from the stored amplitudes and rounded to complex64 when stored --
    the full-state oracle for states whose complex128 form exceeds host memory (c4, n = 34:
    128 GiB).  Pinned against run() in tests/test_oracle.py."""
    n = circuit.n
    psi = np.empty(1 << n, dtype=np.complex64)
    arr, keep = _marshal(circuit.gates)
    rc = lib().oracle_run_c64store(n, circuit.x0, psi.ctypes.data, arr, len(circuit.gates), nthreads)
    if rc != 0:
        raise ValueError(f"oracle: rc={rc}")
    return psi


def norm(psi: np.ndarray) -> float:
    n = int(psi.size).bit_length() - 1
    return lib().oracle_norm(n, np.ascontiguousarray(psi, dtype=np.complex128).ctypes.data)


def padded(n: int, name: str, qs, params=()) -> np.ndarray:
    """Level 2 building block: gate padded to 2^n x 2^n by its definition
    M[i][j] = U[l(i)][l(j)] if i, j agree off the gate's bits, else 0
    (PAPER.md L230-233)."""
    U = gate_matrix(name, params)
    q = len(qs)
    N = 1 << n
    idx = np.arange(N)
    loc = np.zeros(N, dtype=np.int64)
    for i, qq in enumerate(qs):
        loc |= ((idx >> qq) & 1) << (q - 1 - i)
    mask = 0
    for qq in qs:
        mask |= 1 << qq
    off = idx & ~mask
    same = off[:, None] == off[None, :]
    return np.where(same, U[loc[:, None], loc[None, :]], 0)


def kron_unitary(n: int, gates) -> np.ndarray:
    """Level 2 (n <= 8): the whole circuit as one dense matrix."""
    assert n <= 8
    M = np.eye(1 << n, dtype=np.complex128)
    for name, qs, p in gates:
        M = padded(n, name, qs, p) @ M
    return M


def compare(psi: np.ndarray, ref: np.ndarray, chunk: int = 1 << 26) -> dict:
    """max_abs, fidelity F = |<ref|psi>|^2/(|ref|^2|psi|^2),
    both norms; streamed in fixed-order chunks, fp64."""
    assert psi.size == ref.size
    max_abs = 0.0
    ov = 0j
    n1 = n2 = 0.0
    for s in range(0, psi.size, chunk):
        a = np.asarray(psi[s:s + chunk], dtype=np.complex128)
        b = np.asarray(ref[s:s + chunk], dtype=np.complex128)
        max_abs = max(max_abs, float(np.max(np.abs(a - b))) if a.size else 0.0)
        ov += np.vdot(b, a)
        n1 += float(np.vdot(a, a).real)
        n2 += float(np.vdot(b, b).real)
    fid = abs(ov) ** 2 / (n1 * n2) if n1 > 0 and n2 > 0 else 0.0
    n = int(psi.size).bit_length() - 1
    return {"max_abs": max_abs, "fidelity": fid, "norm_gpu": n1, "norm_ref": n2,
            "max_abs_rms": max_abs * 2 ** (n / 2)}


def timed_run(circuit, nthreads: int = 0, gates=None):
    t0 = time.perf_counter()
    psi = run(circuit, nthreads, gates)
    return psi, time.perf_counter() - t0


# ---------------------------------------------------------------------------
# One amplitude at a time, for circuits of monomial gates (sampled parity at
# full size, VERDICT r1 / SURVEY.md 8(c) "sampled outputs the oracle can compute
# one by one").  (U psi)[y] = sum_x U[y, x] psi[x] (one row of
# the padded matrix); when every row of every gate matrix has exactly one
# nonzero entry (X, CNOT, SWAP, Z, S, T, CZ, CPHASE: permutations times phases)
# the sum has one term, so psi_out[y] = (product of the entries met while walking
# y back through the gates) * psi_in[x].  Generic in the gate: the nonzero
# entries are read from gate_matrix(), the oracle's own table; plain numpy over
# an array of indices, no special case per gate kind.
# ---------------------------------------------------------------------------
def monomial_amplitudes(n: int, gates, psi_in, ys) -> np.ndarray:
    """psi_out[ys] for psi_out = U_G ... U_1 psi_in, every U_g monomial; psi_in is a
    callable mapping an array of indices to their input amplitudes."""
    idx = np.array(ys, dtype=np.uint64)
    amp = np.ones(idx.size, dtype=np.complex128)
    for name, qs, p in reversed(list(gates)):
        U = gate_matrix(name, p)
        d, q = U.shape[0], len(qs)
        col = np.empty(d, dtype=np.int64)
        for r in range(d):
            nz = np.flatnonzero(U[r] != 0)
            if nz.size != 1:
                raise ValueError(f"{name} is not monomial")
            col[r] = nz[0]
        ent = U[np.arange(d), col]
        row = np.zeros(idx.size, dtype=np.int64)
        for i, qq in enumerate(qs):            # first-listed qubit = MSB of the local index
            row |= ((idx >> np.uint64(qq)) & np.uint64(1)).astype(np.int64) << (q - 1 - i)
        amp *= ent[row]
        c = col[row]
        for i, qq in enumerate(qs):
            bit = ((c >> (q - 1 - i)) & 1).astype(np.uint64)
            idx = (idx & ~np.uint64(1 << qq)) | (bit << np.uint64(qq))
    return amp * psi_in(idx)


def qft_basis_amplitudes(n: int, x0: int, ys) -> np.ndarray:
    """QFT of |x0> at indices ys (reading A7, pinned against run() for n = 3..10):
    2^{-n/2} exp(2 pi i ((x0 y) mod 2^n) / 2^n), the product reduced exactly in
    integers before the single rounding to double."""
    y = np.asarray(ys, dtype=np.uint64)
    if n <= 32:
        r = (np.uint64(x0) * y) & np.uint64((1 << n) - 1)        # < 2^64: exact
        frac = r.astype(np.float64) / float(1 << n)
    else:
        frac = np.array([((x0 * int(v)) % (1 << n)) / float(1 << n) for v in y])
    return 2.0 ** (-n / 2) * np.exp(2j * np.pi * frac)


# ---------------------------------------------------------------------------
# Measurement sampling ("Simulating
# measurements is then straightforward").  The definition,
# written out: the s-th draw takes u_s from the (s+1)-th output of splitmix64
# seeded with `seed`, u_s = (out >> 11) * 2^-53, and returns the first LOGICAL index j
# at which the fp64 cumulative sum of |a|^2 (in logical order) exceeds
# u_s * total (inverse-CDF sampling; Born rule).  Plain numpy, no blocking.
# ---------------------------------------------------------------------------
_GAMMA = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1


def splitmix64(seed: int, s: int) -> int:
    """(s+1)-th output of Vigna's splitmix64 seeded with `seed`."""
    z = (seed + (s + 1) * _GAMMA) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def uniforms(seed: int, shots: int) -> np.ndarray:
    return np.array([(splitmix64(seed, s) >> 11) * 2.0 ** -53 for s in range(shots)], dtype=np.float64)


def sample(psi: np.ndarray, seed: int, shots: int) -> np.ndarray:
    """Inverse-CDF samples of |psi|^2 in logical index order (Born rule)."""
    prob = np.abs(np.asarray(psi, dtype=np.complex128)) ** 2
    cdf = np.cumsum(prob)                      # sequential, logical order
    total = cdf[-1]
    u = uniforms(seed, shots) * total
    idx = np.searchsorted(cdf, u, side="right")  # first j with cdf[j] > u
    idx = np.minimum(idx, prob.size - 1)
    return idx.astype(np.uint64)
