"""CPU emulator of the encoded device plan blob (tests only).

Decodes the exact bytes the kernels read (`sv_plan_blob`, layout of
paper_2008_00216_b200/csrc/pass_format.h) and applies every op / group
sub-op to a numpy complex128 state using the physical bit each field names.
Passing here while a GPU parity test fails localises a bug to the kernel
rather than the planner or the encoder.  Shares no code with oracle/.
"""
import ctypes as ct

import numpy as np

from tests import plan_interp as PI

MAXT = 14


class Term(ct.Structure):
    _fields_ = [("a", ct.c_int32), ("b", ct.c_int32), ("ang", ct.c_uint64)]


class Diag(ct.Structure):
    _fields_ = [("cst", ct.c_uint64), ("lin", ct.c_uint64 * MAXT), ("A", (ct.c_uint64 * MAXT) * MAXT),
                ("n_cross", ct.c_int32), ("n_olin", ct.c_int32), ("n_oquad", ct.c_int32), ("all_quarter", ct.c_int32),
                ("cross_off", ct.c_uint32), ("olin_off", ct.c_uint32), ("oquad_off", ct.c_uint32), ("pad", ct.c_uint32),
                ("cross_start", ct.c_int32 * (MAXT + 2))]


class Op(ct.Structure):
    _fields_ = [("type", ct.c_int32), ("k", ct.c_int32), ("tpos", ct.c_int32 * 6), ("mat_off", ct.c_uint32),
                ("t_loc", ct.c_int32), ("c_loc", ct.c_int32), ("c_phys", ct.c_int32), ("diag_off", ct.c_uint32),
                ("nsub", ct.c_int32), ("sub_off", ct.c_uint32), ("pad", ct.c_int32)]


class Sub(ct.Structure):
    _fields_ = [("code", ct.c_int32), ("arg", ct.c_uint32), ("ctl", ct.c_uint32), ("pad", ct.c_uint32)]


class Group(ct.Structure):
    _fields_ = [("nsub", ct.c_int32), ("sub_off", ct.c_uint32), ("nvb", ct.c_int32), ("pair16", ct.c_int32),
                ("tpos", ct.c_int32 * 4), ("sw_off", ct.c_uint32 * 16), ("vbit", (ct.c_uint32 * 2) * (MAXT - 4)),
                ("vtab_off", ct.c_uint32), ("nflip_g", ct.c_int32), ("nflip_s", ct.c_int32), ("pad", ct.c_int32),
                ("flip", ct.c_uint32 * 16)]


class DTab(ct.Structure):
    _fields_ = [("stat_off", ct.c_uint32), ("cstat_off", ct.c_uint32), ("term_off", ct.c_uint32),
                ("nterm", ct.c_int32), ("m", ct.c_int32), ("ent_off", ct.c_uint32), ("half", ct.c_int32),
                ("vraw", ct.c_uint16 * 6), ("pad2", ct.c_uint32 * 2)]


class Pass(ct.Structure):
    _fields_ = [("kind", ct.c_int32), ("S", ct.c_int32), ("L", ct.c_int32), ("h", ct.c_int32),
                ("hpos", ct.c_int32 * MAXT), ("out_mask", ct.c_uint64), ("rank_bits", ct.c_uint64),
                ("n_local", ct.c_int32), ("nops", ct.c_int32), ("ops_off", ct.c_uint32), ("mat_off", ct.c_uint32),
                ("mat_bytes", ct.c_uint32), ("cnot_c", ct.c_int32), ("cnot_t", ct.c_int32), ("diag_off", ct.c_uint32),
                ("rec_bytes", ct.c_uint32), ("ntab", ct.c_int32), ("tab_off", ct.c_uint32), ("grouped", ct.c_int32),
                ("tab_entries", ct.c_uint32), ("param_bytes", ct.c_uint32),
                ("tc_off", ct.c_uint32), ("ntc", ct.c_int32), ("ntcop", ct.c_int32), ("swz_tma", ct.c_int32),
                ("tperm", ct.c_uint8 * 48)]


class TcStep(ct.Structure):
    _fields_ = [("kind", ct.c_int16), ("last", ct.c_int16), ("first", ct.c_int16), ("n", ct.c_int16),
                ("op", ct.c_int32), ("group", ct.c_int32), ("dep", ct.c_uint64), ("bvar", ct.c_int32), ("pad", ct.c_int32)]


assert ct.sizeof(Op) == 64 and ct.sizeof(Sub) == 16 and ct.sizeof(Pass) == 208 and ct.sizeof(Term) == 16
assert ct.sizeof(Group) == 256 and ct.sizeof(DTab) == 48 and ct.sizeof(TcStep) == 32

U2_PAIRS = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


def _at(blob, cls, off):
    return cls.from_buffer_copy(blob, off)


def _terms(blob, off, n):
    return [_at(blob, Term, off + 16 * i) for i in range(n)]


def _bits(j, p):
    return (j >> np.uint64(p)) & np.uint64(1)


def _phase_apply(psi, ph):
    hi = (ph >> np.uint64(32)).astype(np.float64)
    lo = (ph & np.uint64(0xFFFFFFFF)).astype(np.float64)
    return psi * np.exp(2j * np.pi * (hi * 2.0 ** 32 + lo) / 2.0 ** 64)


def _matrix(blob, off, D, c128):
    if c128:
        a = np.frombuffer(blob, dtype=np.float64, count=2 * D * D, offset=off)
    else:
        a = np.frombuffer(blob, dtype=np.float32, count=2 * D * D, offset=off).astype(np.float64)
    return (a[0::2] + 1j * a[1::2]).reshape(D, D)


def _matrix_packed(blob, off, D, c128):
    """Group sub-op matrix: complex128 interleaved; complex64 re[D*D] then (-im, im) pairs."""
    if c128:
        return _matrix(blob, off, D, True)
    re = np.frombuffer(blob, dtype=np.float32, count=D * D, offset=off).astype(np.float64)
    pr = np.frombuffer(blob, dtype=np.float32, count=2 * D * D, offset=off + 4 * D * D).astype(np.float64)
    assert np.all(pr[0::2] == -pr[1::2])
    return (re + 1j * pr[1::2]).reshape(D, D)


def run(n, blob, offs, x0=0, c128=False):
    psi = np.zeros(1 << n, dtype=np.complex128)
    psi[x0] = 1
    j = np.arange(1 << n, dtype=np.uint64)
    for po in offs:
        P = _at(blob, Pass, po)
        if P.kind == 4:
            raise NotImplementedError("remaps are executed host-side; use n_global=0")
        if P.kind == 3:
            psi = PI._cnot(psi, n, P.cnot_c, P.cnot_t)
            continue
        pos2phys = [i for i in range(P.L)] + [P.hpos[r] for r in range(P.h)]
        if P.kind == 2:
            ops = [("diag", P.diag_off)]
        elif P.grouped:
            ops = [("group", _at(blob, Group, po + P.ops_off + ct.sizeof(Group) * i)) for i in range(P.nops)]
        else:
            ops = [("op", _at(blob, Op, po + P.ops_off + 64 * i)) for i in range(P.nops)]
        with np.errstate(over="ignore"):
            for kind, op in ops:
                if kind == "group":
                    psi = _run_group(psi, n, blob, po, P, op, pos2phys, c128, j)
                elif kind == "diag" or op.type == 2:
                    doff = po + (op if kind == "diag" else op.diag_off)
                    D = _at(blob, Diag, doff)
                    ph = np.full(1 << n, np.uint64(D.cst), dtype=np.uint64)
                    for q in range(P.S):
                        ph += _bits(j, pos2phys[q]) * np.uint64(D.lin[q])
                        for r in range(q + 1, P.S):
                            ph += _bits(j, pos2phys[q]) * _bits(j, pos2phys[r]) * np.uint64(D.A[q][r])
                    for t in _terms(blob, doff + D.cross_off, D.n_cross):
                        ph += _bits(j, pos2phys[t.a]) * _bits(j, t.b) * np.uint64(t.ang)
                    for t in _terms(blob, doff + D.olin_off, D.n_olin):
                        ph += _bits(j, t.a) * np.uint64(t.ang)
                    for t in _terms(blob, doff + D.oquad_off, D.n_oquad):
                        ph += _bits(j, t.a) * _bits(j, t.b) * np.uint64(t.ang)
                    psi = _phase_apply(psi, ph)
                elif op.type == 1:
                    tg = [pos2phys[op.tpos[i]] for i in range(op.k)]
                    M = _matrix(blob, po + P.mat_off + op.mat_off, 1 << op.k, c128)
                    psi = PI._apply_dense(psi, n, tg, M)
                elif op.type == 3:
                    c = pos2phys[op.c_loc] if op.c_loc >= 0 else op.c_phys
                    psi = PI._cnot(psi, n, c, pos2phys[op.t_loc])
    return psi


def _run_group(psi, n, blob, po, P, g, pos2phys, c128, j):
    """Apply one encoded gate group: local bit k <-> tile position tpos[k]."""
    G = [pos2phys[g.tpos[i]] for i in range(4)]
    assert len(set(g.sw_off[l] for l in range(16))) == 16

    # inverse of the swizzle on single tile positions: flipped position from its swizzled offset
    c128_ = c128
    tma = bool(getattr(P, "swz_tma", 0))

    def swz(i):
        H = [1, 2, 4, 0, 0, 0, 0, 0, 0, 0, 0] if tma else [3, 5, 6, 7, 1, 2, 4, 3, 5, 6, 7]
        def h(x):
            r, j = 0, 0
            while x:
                if x & 1:
                    r ^= H[j]
                x >>= 1
                j += 1
            return r
        if c128_:
            return i ^ h(i >> 3)
        c = i >> 1
        return ((c ^ h(c >> 3)) << 1) | (i & 1)
    pos_of = {swz(1 << q): q for q in range(P.S)}

    def flips(psi, first, cnt):
        for q in range(cnt):
            f = g.flip[first + q]
            tpos, a = pos_of[f & 0xFFFF], f >> 17
            ctl = a if f & (1 << 16) else pos2phys[a.bit_length() - 1]
            assert f & (1 << 16) or (a & (a - 1)) == 0
            psi = PI._cnot(psi, n, ctl, pos2phys[tpos])
        return psi

    psi = flips(psi, 0, g.nflip_g)
    for k in range(g.nsub):
        sb = _at(blob, Sub, po + g.sub_off + 16 * k)
        c = sb.code & 0xFF
        ctl_raw, ctl_phys = sb.ctl & 0xFFFF, (sb.ctl >> 16) - 1
        if c < 4:
            psi = PI._apply_dense(psi, n, [G[c]], _matrix(blob, po + P.mat_off + sb.arg, 2, c128))
        elif c < 10:
            a, b = U2_PAIRS[c - 4]
            psi = PI._apply_dense(psi, n, [G[a], G[b]], _matrix(blob, po + P.mat_off + sb.arg, 4, c128))
        elif 31 <= c < 37:
            a, b = U2_PAIRS[c - 31]
            outbits = [b_ for b_ in range(64) if (P.out_mask >> b_) & 1]
            sel = []
            for i in range(3):
                code = (sb.code >> (8 + 5 * i)) & 31
                if code != 31:
                    sel.append(outbits[code])                  # tile-ordinal bit -> physical bit
            assert all(s_ not in pos2phys for s_ in sel)      # selectors are outside the tile
            esz = 16 if c128 else 8
            jj = np.arange(1 << n)
            out = np.zeros_like(psi)
            for v in range(1 << len(sel)):
                M = _matrix(blob, po + P.mat_off + sb.arg + v * 16 * esz, 4, c128)
                m = np.ones(1 << n, dtype=bool)
                for i, s_ in enumerate(sel):
                    m &= ((jj >> s_) & 1) == ((v >> i) & 1)
                out[m] = PI._apply_dense(psi, n, [G[a], G[b]], M)[m]
            psi = out
        elif 10 <= c < 30:
            cl, t = (c - 10) // 4 - 1, (c - 10) % 4
            ctl = []
            if cl >= 0:
                ctl.append(G[cl])
            if ctl_raw:
                q = ctl_raw.bit_length() - 1
                assert q not in [g.tpos[i] for i in range(4)]   # must be fixed within the vector
                ctl.append(pos2phys[q])
            if ctl_phys >= 0:
                ctl.append(ctl_phys)
            assert len(ctl) <= 1
            if ctl:
                psi = PI._cnot(psi, n, ctl[0], G[t])
            else:
                psi = psi[np.arange(1 << n) ^ (1 << G[t])]
        elif 44 <= c < 54:
            D_ = 2 if c < 48 else 4
            dt = np.float64 if c128 else np.float32
            M = np.frombuffer(blob, dtype=dt, count=D_ * D_, offset=po + P.mat_off + sb.arg).astype(np.float64)
            M = M.reshape(D_, D_).astype(np.complex128)
            tg = [G[c - 44]] if c < 48 else [G[q] for q in U2_PAIRS[c - 48]]
            psi = PI._apply_dense(psi, n, tg, M)
        elif 41 <= c < 44:
            pairs = [((0, 1), (2, 3)), ((0, 2), (1, 3)), ((0, 3), (1, 2))][c - 41]
            outbits = [b_ for b_ in range(64) if (P.out_mask >> b_) & 1]
            esz = 16 if c128 else 8
            jj = np.arange(1 << n)
            for (a, b), off, w in ((pairs[0], sb.arg, sb.code >> 8), (pairs[1], sb.ctl, sb.pad)):
                sel = [outbits[(w >> (5 * i)) & 31] for i in range(3) if ((w >> (5 * i)) & 31) != 31]
                out = np.zeros_like(psi)
                for v in range(1 << len(sel)):
                    M = _matrix(blob, po + P.mat_off + off + v * 16 * esz, 4, c128)
                    m = np.ones(1 << n, dtype=bool)
                    for i, s_ in enumerate(sel):
                        m &= ((jj >> s_) & 1) == ((v >> i) & 1)
                    out[m] = PI._apply_dense(psi, n, [G[a], G[b]], M)[m]
                psi = out
        elif 37 <= c < 41:
            jb = c - 37                                       # half table on local bit jb
            d = _at(blob, DTab, po + P.tab_off + ct.sizeof(DTab) * sb.arg)
            assert d.half == 1
            vq = [d.vraw[i].bit_length() - 1 for i in range(d.m)]
            assert all(q not in [g.tpos[i] for i in range(4)] for q in vq)
            stat = np.frombuffer(blob, dtype=np.uint64, count=8 << d.m, offset=po + d.stat_off)
            e = np.zeros(1 << n, dtype=np.uint64)
            others = [k2 for k2 in range(4) if k2 != jb]
            for i, k2 in enumerate(others):
                e |= _bits(j, G[k2]) << np.uint64(i)
            for i, q in enumerate(vq):
                e |= _bits(j, pos2phys[q]) << np.uint64(3 + i)
            ph = stat[e.astype(np.int64)].copy()
            for t in _terms(blob, po + d.term_off, d.nterm):
                assert t.a < 0                                # per-tile terms are constants
                on = _bits(j, t.b)
                if t.a <= -2:
                    on = on * _bits(j, -2 - t.a)
                ph += on * np.uint64(t.ang)
            ph = ph * _bits(j, G[jb])                          # amplitudes with l_j = 0 unchanged
            psi = _phase_apply(psi, ph)
        else:
            assert c == 30
            d = _at(blob, DTab, po + P.tab_off + ct.sizeof(DTab) * sb.arg)
            vq = [d.vraw[i].bit_length() - 1 for i in range(d.m)]
            assert all(q not in [g.tpos[i] for i in range(4)] for q in vq)
            assert all(d.vraw[i] == 0 for i in range(d.m, 3))
            stat = np.frombuffer(blob, dtype=np.uint64, count=16 << d.m, offset=po + d.stat_off)
            e = np.zeros(1 << n, dtype=np.uint64)
            for k2 in range(4):
                e |= _bits(j, G[k2]) << np.uint64(k2)
            for i, q in enumerate(vq):
                e |= _bits(j, pos2phys[q]) << np.uint64(4 + i)
            ph = stat[e.astype(np.int64)].copy()
            for t in _terms(blob, po + d.term_off, d.nterm):
                on = _bits(j, t.b)
                if t.a >= 0:
                    on = on * ((e >> np.uint64(t.a)) & np.uint64(1))
                elif t.a <= -2:
                    on = on * _bits(j, -2 - t.a)
                ph += on * np.uint64(t.ang)
            psi = _phase_apply(psi, ph)
    return flips(psi, 8, g.nflip_s)
