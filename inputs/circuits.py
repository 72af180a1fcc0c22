"""Seeded synthetic circuit generators shared by the oracle and the CUDA path.

This module holds NO arithmetic of the simulation method: it only draws gate
names, qubit indices and angle parameters (as exact rationals of pi) from a
counter-based generator.  Both `oracle/` and the product binding consume the
resulting gate lists and build their own matrices independently.

Sources:
  * Workloads: BASELINE.json configs[0..4] (c1..c5); the paper's Google v2
    supremacy circuits are not in the container and
    are NOT reproduced -- these seeded circuits stand in for them (DESIGN.md
    "Input recipe").
  * Readings A11-A15 of SURVEY.md 8(c) (cycle structure, gate non-repetition,
    coupler patterns, removed grid sites, c3 tail), listed in DESIGN.md.
  * Draw order: SURVEY.md 8(d) "Draw order".

A gate is a tuple ``(name, qubits, params)``:
  name    one of GATE_NAMES
  qubits  tuple of 1 or 2 distinct ints (first-listed qubit = MSB of the
          gate's local index, PAPER.md L148 CNOT matrix; reading A2)
  params  tuple of angles, each an exact rational multiple of pi given as
          (num, den) -> angle = num*pi/den; for 'u1'/'u2' params is a flat
          tuple of 2*4^q floats (row-major re, im) instead.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

GATE_NAMES = ("h", "x", "y", "z", "s", "t", "sx", "sy", "sw",
              "cz", "cnot", "swap", "cphase", "fsim", "u1", "u2")
ONE_QUBIT = {"h", "x", "y", "z", "s", "t", "sx", "sy", "sw", "u1"}
TWO_QUBIT = {"cz", "cnot", "swap", "cphase", "fsim", "u2"}

Gate = Tuple[str, Tuple[int, ...], tuple]

MASK64 = (1 << 64) - 1


class SplitMix64:
    """splitmix64 (Steele, Lea, Flood 2014) -- the counter-based generator both
    sides share (seed = config number)."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def u(self, m: int) -> int:
        """uniform-ish in [0, m): next() % m (bias <= m/2^64, deterministic)."""
        return self.next() % m


@dataclass
class Circuit:
    name: str
    n: int
    gates: List[Gate]
    x0: int = 0                      # initial computational basis state |x0>
    seed: int = 0
    meta: dict = field(default_factory=dict)

    def text(self) -> str:
        return to_text(self)

    def sha256(self) -> str:
        return hashlib.sha256(self.text().encode()).hexdigest()


# ----------------------------------------------------------------------------
# grid layouts (reading A13, A14)
# ----------------------------------------------------------------------------
_REMOVAL_ORDER = lambda R, C: [(0, 0), (R - 1, C - 1), (0, C - 1), (R - 1, 0), (0, 1)]


def grid_sites(R: int, C: int, removed: int = 0):
    """Kept sites of an R x C grid, the first `removed` sites of the fixed
    removal order dropped; qubits numbered row-major over kept sites (A14)."""
    drop = set(_REMOVAL_ORDER(R, C)[:removed])
    sites = [(r, c) for r in range(R) for c in range(C) if (r, c) not in drop]
    return {s: i for i, s in enumerate(sites)}


def coupler_patterns(R: int, C: int, removed: int = 0):
    """8 alternating coupler classes in order H00, V00, H11, V11, H01, V01,
    H10, V10 (A13).  H_{a,b}: horizontal (r,c)-(r,c+1) with c%2==a, r%2==b;
    V_{a,b}: vertical (r,c)-(r+1,c) with r%2==a, c%2==b.  Each class is a
    matching; pairs are (a<b) ascending."""
    idx = grid_sites(R, C, removed)
    order = [("H", 0, 0), ("V", 0, 0), ("H", 1, 1), ("V", 1, 1),
             ("H", 0, 1), ("V", 0, 1), ("H", 1, 0), ("V", 1, 0)]
    pats = []
    for kind, a, b in order:
        pairs = []
        for (r, c), q in idx.items():
            if kind == "H":
                other = (r, c + 1)
                ok = (c % 2 == a) and (r % 2 == b)
            else:
                other = (r + 1, c)
                ok = (r % 2 == a) and (c % 2 == b)
            if ok and other in idx:
                p = idx[other]
                pairs.append((min(q, p), max(q, p)))
        pats.append(sorted(pairs))
    return pats


_ONEQ = ("sx", "sy", "sw")


def grid_circuit(name: str, R: int, C: int, removed: int, cycles: int,
                 twoq: str, seed: int) -> Circuit:
    """Random grid circuit (BASELINE.json configs c1, c2, c4, c5; A11-A13):
    cycle t = one of {sqrt X, sqrt Y, sqrt W} on every qubit (never repeating
    the qubit's previous gate) then the 2q gate on pattern t mod 8 couplers."""
    idx = grid_sites(R, C, removed)
    n = len(idx)
    pats = coupler_patterns(R, C, removed)
    rng = SplitMix64(seed)
    prev = [None] * n
    gates: List[Gate] = []
    for t in range(cycles):
        for q in range(n):
            if t == 0:
                g = _ONEQ[rng.u(3)]
            else:
                choices = [x for x in _ONEQ if x != prev[q]]
                g = choices[rng.u(2)]
            prev[q] = g
            gates.append((g, (q,), ()))
        for (a, b) in pats[t % 8]:
            if twoq == "cz":
                gates.append(("cz", (a, b), ()))
            elif twoq == "fsim":
                # fSim(theta=pi/2, phi=pi/6)
                gates.append(("fsim", (a, b), ((1, 2), (1, 6))))
            else:
                raise ValueError(twoq)
    return Circuit(name=name, n=n, gates=gates, x0=0, seed=seed,
                   meta={"R": R, "C": C, "removed": removed, "cycles": cycles})


def qft_gates(n: int) -> List[Gate]:
    """QFT in LSB order (reading A7): for j=1..n: H on bit n-j; for k=2..n-j+1:
    R_k = CPHASE(2 pi / 2^k) on bits (n-j-k+1, n-j); then SWAP (n-j, j-1) for
    j <= n/2.  R_k angle = 2 pi / 2^k = pi * 2 / 2^k."""
    gates: List[Gate] = []
    for j in range(1, n + 1):
        gates.append(("h", (n - j,), ()))
        for k in range(2, n - j + 2):
            gates.append(("cphase", (n - j - k + 1, n - j), ((2, 1 << k),)))
    for j in range(1, n // 2 + 1):
        gates.append(("swap", (n - j, j - 1), ()))
    return gates


def qft_circuit(n: int = 32, tail: int = 200, seed: int = 3, name: str = "c3") -> Circuit:
    """BASELINE.json configs[2] (c3): QFT on a seeded basis state |x0> followed
    by `tail` random CNOT/X/CZ/T gates (reading A15)."""
    rng = SplitMix64(seed)
    x0 = rng.next() & ((1 << min(n, 32)) - 1) if n <= 32 else rng.next() & MASK64 & ((1 << n) - 1)
    gates = qft_gates(n)
    for _ in range(tail):
        ty = rng.u(4)
        if ty in (0, 2):
            a = rng.u(n)
            b = rng.u(n - 1)
            b += (b >= a)
            gates.append((("cnot", "cz")[ty // 2], (a, b), ()))
        else:
            q = rng.u(n)
            gates.append((("x", "t")[ty // 2], (q,), ()))
    return Circuit(name=name, n=n, gates=gates, x0=x0, seed=seed, meta={"tail": tail})


def config(c: int, n_override: int | None = None) -> Circuit:
    """The five BASELINE.json configs as seeded synthetic circuits."""
    if c == 1:
        return grid_circuit("c1", 4, 4, 0, 20, "cz", 1)
    if c == 2:
        return grid_circuit("c2", 5, 6, 0, 20, "fsim", 2)
    if c == 3:
        return qft_circuit(32 if n_override is None else n_override, 200, 3)
    if c == 4:
        return grid_circuit("c4", 6, 6, 2, 14, "fsim", 4)
    if c == 5:
        return grid_circuit("c5", 6, 7, 5, 14, "fsim", 5)
    raise ValueError(c)


def weak_ladder(n: int) -> Circuit:
    """Weak-scaling ladder n=34/35/36/37 (seed 5, 14 cycles; A14)."""
    shapes = {34: (6, 6, 2), 35: (6, 6, 1), 36: (6, 6, 0), 37: (6, 7, 5)}
    R, C, rm = shapes[n]
    return grid_circuit(f"weak{n}", R, C, rm, 14, "fsim", 5)


# ----------------------------------------------------------------------------
# generic random circuits for parity tests (all gate kinds)
# ----------------------------------------------------------------------------
def random_unitary(dim: int, rng: SplitMix64) -> tuple:
    """Haar-ish random unitary from seeded Box-Muller Gaussians + Gram-Schmidt
    (input data, not method arithmetic).  Returns flat (re, im) row-major."""
    import math
    def gauss():
        u1 = (rng.next() >> 11) * 2.0 ** -53
        u2 = (rng.next() >> 11) * 2.0 ** -53
        u1 = max(u1, 1e-300)
        return math.sqrt(-2 * math.log(u1)) * math.cos(2 * math.pi * u2)
    cols = []
    for _ in range(dim):
        v = [complex(gauss(), gauss()) for _ in range(dim)]
        for w in cols:
            d = sum(wi.conjugate() * vi for wi, vi in zip(w, v))
            v = [vi - d * wi for vi, wi in zip(v, w)]
        nrm = math.sqrt(sum(abs(x) ** 2 for x in v))
        cols.append([x / nrm for x in v])
    out = []
    for r in range(dim):
        for c in range(dim):
            out += [cols[c][r].real, cols[c][r].imag]
    return tuple(out)


def random_circuit(n: int, ngates: int, seed: int, kinds: Sequence[str] | None = None,
                   x0: int | None = None) -> Circuit:
    """Random circuit over `kinds` (default: every gate kind) on n qubits."""
    rng = SplitMix64(seed * 7919 + 17)
    kinds = list(kinds or GATE_NAMES)
    if n < 2:
        kinds = [k for k in kinds if k in ONE_QUBIT]
    gates: List[Gate] = []
    for _ in range(ngates):
        k = kinds[rng.u(len(kinds))]
        if k in ONE_QUBIT:
            qs = (rng.u(n),)
        else:
            a = rng.u(n)
            b = rng.u(n - 1)
            b += (b >= a)
            qs = (a, b)
        if k == "cphase":
            params = ((int(rng.u(31)) - 15, 1 << rng.u(6)),)
        elif k == "fsim":
            # mix of the relabel-able theta=pi/2 case and generic angles
            th = (1, 2) if rng.u(2) == 0 else (int(rng.u(23)) - 11, 12)
            params = (th, (int(rng.u(23)) - 11, 12))
        elif k == "u1":
            params = random_unitary(2, rng)
        elif k == "u2":
            params = random_unitary(4, rng)
        else:
            params = ()
        gates.append((k, qs, params))
    if x0 is None:
        x0 = rng.next() & ((1 << n) - 1)
    return Circuit(name=f"rand{n}_{ngates}_{seed}", n=n, gates=gates, x0=x0, seed=seed)


def inverse_gates(gates: Sequence[Gate]) -> List[Gate]:
    """Gate list of C^dagger (for the mirror test C^dagger C |x> = |x>):
    reversed order; self-inverse gates kept, every other gate marked adjoint
    by the '_dg' name suffix (both sides apply the conjugate transpose)."""
    inv: List[Gate] = []
    for name, qs, p in reversed(list(gates)):
        if name in ("h", "x", "y", "z", "cz", "cnot", "swap"):
            inv.append((name, qs, p))
        elif name.endswith("_dg"):
            inv.append((name[:-3], qs, p))
        else:
            inv.append((name + "_dg", qs, p))
    return inv


def base_name(name: str) -> Tuple[str, bool]:
    """('sx_dg') -> ('sx', True)."""
    if name.endswith("_dg"):
        return name[:-3], True
    return name, False


# ----------------------------------------------------------------------------
# text format (extends SPEC.md L100's cycle-prefixed format)
# ----------------------------------------------------------------------------
def _fmt_angle(a):
    num, den = a
    return f"{num}*pi/{den}"


def to_text(c: Circuit) -> str:
    lines = [f"# config={c.name} n={c.n} seed={c.seed} x0={c.x0}"]
    for i, (name, qs, p) in enumerate(c.gates):
        s = f"{i} {name} " + " ".join(str(q) for q in qs)
        if base_name(name)[0] in ("u1", "u2"):
            s += " " + " ".join(repr(float(x)) for x in p)
        elif p:
            s += " " + " ".join(_fmt_angle(a) for a in p)
        lines.append(s)
    return "\n".join(lines) + "\n"


def from_text(text: str) -> Circuit:
    head, *body = [l for l in text.splitlines() if l.strip()]
    kv = dict(tok.split("=") for tok in head[1:].split())
    gates: List[Gate] = []
    for line in body:
        toks = line.split()
        name = toks[1]
        nq = 1 if base_name(name)[0] in ONE_QUBIT else 2
        qs = tuple(int(t) for t in toks[2:2 + nq])
        rest = toks[2 + nq:]
        if base_name(name)[0] in ("u1", "u2"):
            p = tuple(float(x) for x in rest)
        else:
            p = tuple((int(a.split("*")[0]), int(a.split("/")[1])) for a in rest)
        gates.append((name, qs, p))
    return Circuit(name=kv["config"], n=int(kv["n"]), gates=gates,
                   x0=int(kv["x0"]), seed=int(kv["seed"]))
