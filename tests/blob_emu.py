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
    _fields_ = [("type", ct.c_int32), ("a", ct.c_int32), ("b", ct.c_int32), ("c_tile", ct.c_int32),
                ("c_phys", ct.c_int32), ("mat_off", ct.c_uint32), ("gdiag_off", ct.c_uint32), ("tbl", ct.c_int32)]


class GDiag(ct.Structure):
    _fields_ = [("cst", ct.c_uint64), ("w", ct.c_uint64 * 4), ("A", (ct.c_uint64 * 4) * 4),
                ("n_cross", ct.c_int32), ("n_olin", ct.c_int32), ("n_oquad", ct.c_int32), ("n_v", ct.c_int32),
                ("cross_off", ct.c_uint32), ("olin_off", ct.c_uint32), ("oquad_off", ct.c_uint32), ("pad2", ct.c_uint32),
                ("n_vlin", ct.c_int32), ("n_vquad", ct.c_int32), ("n_vcross", ct.c_int32), ("n_vout", ct.c_int32),
                ("vlin_off", ct.c_uint32), ("vquad_off", ct.c_uint32), ("vcross_off", ct.c_uint32), ("vout_off", ct.c_uint32)]


class Pass(ct.Structure):
    _fields_ = [("kind", ct.c_int32), ("S", ct.c_int32), ("L", ct.c_int32), ("h", ct.c_int32),
                ("hpos", ct.c_int32 * MAXT), ("out_mask", ct.c_uint64), ("rank_bits", ct.c_uint64),
                ("n_local", ct.c_int32), ("nops", ct.c_int32), ("ops_off", ct.c_uint32), ("mat_off", ct.c_uint32),
                ("mat_bytes", ct.c_uint32), ("cnot_c", ct.c_int32), ("cnot_t", ct.c_int32), ("diag_off", ct.c_uint32),
                ("rec_bytes", ct.c_uint32), ("ntab", ct.c_int32), ("tab_off", ct.c_uint32), ("pad2", ct.c_int32 * 3)]


assert ct.sizeof(Op) == 64 and ct.sizeof(Sub) == 32 and ct.sizeof(Pass) == 144 and ct.sizeof(Term) == 16


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
        else:
            ops = [("op", _at(blob, Op, po + P.ops_off + 64 * i)) for i in range(P.nops)]
        with np.errstate(over="ignore"):
            for kind, op in ops:
                if kind == "diag" or op.type == 2:
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
                elif op.type == 4:
                    G = [pos2phys[op.tpos[i]] for i in range(4)]
                    for k in range(op.nsub):
                        sb = _at(blob, Sub, po + op.sub_off + 32 * k)
                        if sb.type == 1:
                            psi = PI._apply_dense(psi, n, [G[sb.a]], _matrix(blob, po + P.mat_off + sb.mat_off, 2, c128))
                        elif sb.type == 2:
                            psi = PI._apply_dense(psi, n, [G[sb.a], G[sb.b]],
                                                  _matrix(blob, po + P.mat_off + sb.mat_off, 4, c128))
                        elif sb.type == 3:
                            goff = po + sb.gdiag_off
                            gd = _at(blob, GDiag, goff)
                            ph = np.full(1 << n, np.uint64(gd.cst), dtype=np.uint64)
                            for t in _terms(blob, goff + gd.olin_off, gd.n_olin):
                                ph += _bits(j, t.a) * np.uint64(t.ang)
                            for t in _terms(blob, goff + gd.oquad_off, gd.n_oquad):
                                ph += _bits(j, t.a) * _bits(j, t.b) * np.uint64(t.ang)
                            for q in range(4):
                                ph += _bits(j, G[q]) * np.uint64(gd.w[q])
                                for r in range(q + 1, 4):
                                    ph += _bits(j, G[q]) * _bits(j, G[r]) * np.uint64(gd.A[q][r])
                            for t in _terms(blob, goff + gd.cross_off, gd.n_cross):
                                ph += _bits(j, G[t.a]) * _bits(j, t.b) * np.uint64(t.ang)
                            tpos = [op.tpos[i] for i in range(4)]
                            for t in _terms(blob, goff + gd.vlin_off, gd.n_vlin):
                                assert t.a not in tpos
                                ph += _bits(j, pos2phys[t.a]) * np.uint64(t.ang)
                            for t in _terms(blob, goff + gd.vquad_off, gd.n_vquad):
                                ph += _bits(j, pos2phys[t.a]) * _bits(j, pos2phys[t.b]) * np.uint64(t.ang)
                            for t in _terms(blob, goff + gd.vcross_off, gd.n_vcross):
                                assert t.b not in tpos
                                ph += _bits(j, G[t.a]) * _bits(j, pos2phys[t.b]) * np.uint64(t.ang)
                            for t in _terms(blob, goff + gd.vout_off, gd.n_vout):
                                ph += _bits(j, pos2phys[t.a]) * _bits(j, t.b) * np.uint64(t.ang)
                            psi = _phase_apply(psi, ph)
                        else:
                            if sb.a >= 0:
                                psi = PI._cnot(psi, n, G[sb.a], G[sb.b])
                            elif sb.c_tile >= 0:
                                # the kernel reads this control from the vector base: it must not
                                # be one of the group's positions (else it varies in the vector)
                                assert sb.c_tile not in [op.tpos[i] for i in range(4)]
                                psi = PI._cnot(psi, n, pos2phys[sb.c_tile], G[sb.b])
                            elif sb.c_phys >= 0:
                                psi = PI._cnot(psi, n, sb.c_phys, G[sb.b])
                            else:
                                t = G[sb.b]
                                psi = psi[np.arange(1 << n) ^ (1 << t)]
    return psi
