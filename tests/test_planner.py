"""Host-side planner tests (-m "not gpu"): the C-ABI library loads without a
GPU, exports every symbol of include/sv.h, and its plans -- executed by an
independent CPU interpreter (tests/plan_interp.py) -- reproduce the oracle.
"""
import os
import re

import numpy as np
import pytest

import oracle
import paper_2008_00216_b200 as stv
from inputs import circuits as C
from tests import plan_interp as PI

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "sv.h")).read()
    declared = set(re.findall(r"^\s*(?:sv_status|const char \*)\s*(sv_\w+)\(", hdr, re.M))
    assert declared == set(stv.EXPORTS)
    L = stv.lib()
    for f in declared:
        assert getattr(L, f) is not None
    assert "sm_100a" in stv.version()


def _check(circ, tol=1e-11, n_global=0, **kw):
    plan = stv.plan_json(circ.n, circ.gates, n_global=n_global, **kw)
    psi = PI.logical(plan, PI.run(plan, x0=circ.x0))
    ref = oracle.run(circ)
    err = np.max(np.abs(psi - ref))
    assert err < tol, (err, kw)
    return plan


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("kmax", [1, 2, 4])
def test_random_all_kinds(seed, kmax):
    circ = C.random_circuit(9, 120, seed)
    _check(circ, kmax=kmax, tile_bits=6, low_bits=2)


@pytest.mark.parametrize("flags", [stv.OPT_NO_RELABEL, stv.OPT_NO_REORDER, stv.OPT_ONE_GATE,
                                   stv.OPT_NO_DIAG_FOLD, stv.OPT_NO_RELABEL | stv.OPT_NO_REORDER])
def test_ablation_flags_preserve_semantics(flags):
    circ = C.random_circuit(8, 150, 11)
    _check(circ, flags=flags, tile_bits=6, low_bits=2)


@pytest.mark.parametrize("tile_bits,low_bits", [(2, 0), (3, 1), (5, 3), (8, 5), (12, 5)])
def test_tile_shapes(tile_bits, low_bits):
    circ = C.random_circuit(10, 100, 3)
    _check(circ, tile_bits=tile_bits, low_bits=low_bits)


def test_c1_config_plan():
    circ = C.config(1)
    plan = _check(circ, tol=1e-10)
    # every non-relabel gate absorbed exactly once
    absorbed = [g for ps in plan["passes"] for g in ps["gates"]]
    assert len(absorbed) == len(set(absorbed)) == len(circ.gates)
    # fusion reduced the 380 gates to far fewer passes
    assert len(plan["passes"]) < len(circ.gates) // 4


def test_qft_and_tail():
    circ = C.qft_circuit(10, tail=120, seed=3)
    plan = _check(circ, tol=1e-10)
    srcs = {g for ps in plan["passes"] for g in ps["gates"]}
    names = [g[0] for g in circ.gates]
    # SWAPs and X are relabels: never part of a pass
    assert all(names[i] not in ("swap", "x") for i in srcs)


def test_grid_fsim_relabel():
    circ = C.grid_circuit("g", 3, 3, 0, 8, "fsim", 7)
    plan = _check(circ)
    # fSim(pi/2, phi) = SWAP . diag: no dense 2-qubit op is needed for it
    assert all(op["type"] != 1 or len(op["tg"]) <= 4 for ps in plan["passes"] for op in ps["ops"])


@pytest.mark.parametrize("g", [1, 2, 3])
def test_global_qubit_remaps(g):
    circ = C.random_circuit(9, 150, 20 + g)
    plan = _check(circ, n_global=g, tile_bits=5, low_bits=2)
    nl = circ.n - g
    for ps in plan["passes"]:
        if ps["kind"] == 4:
            for gb, lb in ps["swaps"]:
                assert gb >= nl and lb < nl
        else:
            for op in ps["ops"]:          # non-diagonal targets only on local bits
                if op["type"] == 1:
                    assert max(op["tg"]) < nl
                if op["type"] == 3:
                    assert op["t"] < nl
    assert any(ps["kind"] == 4 for ps in plan["passes"])


def test_mirror_plan():
    circ = C.random_circuit(8, 80, 5)
    full = C.Circuit("m", 8, circ.gates + C.inverse_gates(circ.gates), x0=circ.x0)
    plan = stv.plan_json(8, full.gates, tile_bits=6, low_bits=2)
    psi = PI.logical(plan, PI.run(plan, x0=circ.x0))
    e = np.zeros(256, complex)
    e[circ.x0] = 1
    assert np.max(np.abs(psi - e)) < 1e-11


def test_diag_form_matches_paper_masks(golden):
    # the per-qubit CZ masks of PAPER.md L522-527 and the planner's single
    # phase form for the same six CZ gates agree on every basis state
    g = golden["paper_bitmasks"]["cz_complete_graph_4q"]
    masks = [int(s, 2) for s in g["masks"]]
    gates = [("cz", (a, b), ()) for a in range(4) for b in range(a + 1, 4)]
    plan = stv.plan_json(4, gates, tile_bits=2, low_bits=0)
    diag_ops = [op for ps in plan["passes"] for op in ps["ops"]]
    assert len(plan["passes"]) == 1 and len(diag_ops) == 1 and diag_ops[0]["type"] == 2
    ph = PI._phase(4, diag_ops[0])
    for j in range(16):
        cnt = sum(bin(masks[k] & j).count("1") for k in range(4) if j >> k & 1)
        assert abs(ph[j] - (-1 if cnt & 2 else 1)) < 1e-15


def test_validation_errors():
    bad = [("h", (5,), ())]
    with pytest.raises(stv.SvError, match="gate 0"):
        stv.plan_json(4, bad)
    with pytest.raises(stv.SvError, match="duplicate"):
        stv.plan_json(4, [("h", (0,), ()), ("cz", (1, 1), ())])
    with pytest.raises(stv.SvError, match="not unitary"):
        stv.plan_json(4, [("u1", (0,), (1.0, 0, 1.0, 0, 0, 0, 1.0, 0))])


def test_remap_peers_schedule():
    # rank r, swapping global bit b: chunk c goes to r with bit b set to c
    assert stv.remap_peers(1, 0, 0b1, 1) == [0, 1]
    assert stv.remap_peers(1, 1, 0b1, 1) == [0, 1]
    assert stv.remap_peers(3, 5, 0b110, 2) == [1, 3, 5, 7]
    assert stv.remap_peers(2, 2, 0b01, 1) == [2, 3]


def _tile_of(ps):
    return int(ps["S"])


@pytest.mark.parametrize("seed", range(4))
def test_group_structure(seed):
    # register-resident gate groups: non-diagonal targets of every sub-op are
    # among the group's <= 4 register bits, which are tile bits
    circ = C.random_circuit(12, 200, 100 + seed)
    plan = _check(circ, tile_bits=8, low_bits=3, budget=400)
    ngroups = 0
    for ps in plan["passes"]:
        if ps["kind"] != 1:
            continue
        S = _tile_of(ps)
        for op in ps["ops"]:
            if op["type"] != 4:
                continue
            ngroups += 1
            T = int(op["T"])
            assert bin(T).count("1") <= 4 and (T & ~S) == 0
            for so in op["subs"]:
                if so["type"] == 1:
                    assert all((T >> q) & 1 for q in so["tg"])
                elif so["type"] == 3:
                    assert (T >> so["t"]) & 1
                # diagonal sub-ops may also touch in-tile bits outside T ("V-bits",
                # per-vector terms) and bits outside the tile (per-tile terms)
    assert ngroups > 0


def test_groups_vs_flat_ops_same_state():
    circ = C.config(1)
    a = stv.plan_json(circ.n, circ.gates)
    b = stv.plan_json(circ.n, circ.gates, flags=stv.OPT_NO_GROUPS)
    pa = PI.logical(a, PI.run(a, x0=0))
    pb = PI.logical(b, PI.run(b, x0=0))
    assert np.max(np.abs(pa - pb)) < 1e-12


from tests import blob_emu as BE


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("case", ["rand", "opts_tile8", "budget400", "budget20_cnots", "qft_tail", "c1"])
def test_encoded_blob_semantics(case, dtype):
    """The exact device blob, emulated on CPU, reproduces the oracle."""
    kw = {}
    if case == "rand":
        circ = C.random_circuit(11, 200, 7)
    elif case == "opts_tile8":
        circ = C.random_circuit(12, 300, 42)
        kw = dict(tile_bits=8, low_bits=3)
    elif case == "budget400":
        circ = C.random_circuit(12, 300, 42)
        kw = dict(budget=400)
    elif case == "budget20_cnots":
        circ = C.random_circuit(11, 120, 5, kinds=["cnot", "h", "cphase"])
        kw = dict(budget=20)
    elif case == "qft_tail":
        circ = C.qft_circuit(11, tail=200, seed=3)
    else:
        circ = C.config(1)
    blob, offs = stv.plan_blob(circ.n, circ.gates, dtype=dtype, **kw)
    plan = stv.plan_json(circ.n, circ.gates, dtype=dtype, **kw)
    psi = PI.logical(plan, BE.run(circ.n, blob, offs, x0=circ.x0, c128=dtype == "c128"))
    ref = oracle.run(circ)
    tol = 2e-6 if dtype == "c64" else 1e-11
    assert np.max(np.abs(psi - ref)) < tol


def _swz_slot(chunk, tma=False):
    """Shared-memory slot of a 16-B tile chunk (pass_format.h, restated): the group pass's
    kSwzH pattern, or TMA SWIZZLE_128B (chunk j of each 128-B line at j ^ (line mod 8))."""
    H = [1, 2, 4, 0, 0, 0, 0, 0, 0, 0, 0] if tma else [3, 5, 6, 7, 1, 2, 4, 3, 5, 6, 7]
    h, x, j = 0, chunk >> 3, 0
    while x:
        if x & 1:
            h ^= H[j]
        x >>= 1
        j += 1
    return chunk ^ h


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("case", ["c2", "qft", "tile9"])
def test_group_layout_bijective_and_conflict_free(case, dtype):
    """Every group's (vector, local index) -> shared-memory address map is the
    swizzle of the raw tile index, a bijection of the tile; every warp phase of
    the group gathers (8 lanes x 16 B, or 16 lanes x 8 B) hits distinct banks."""
    if case == "c2":
        circ, kw = C.config(2), {}
    elif case == "qft":
        circ, kw = C.qft_circuit(20, tail=100, seed=9), {}
    else:
        circ, kw = C.random_circuit(14, 200, 3), dict(tile_bits=9, low_bits=3)
    blob, offs = stv.plan_blob(circ.n, circ.gates, dtype=dtype, **kw)
    c128 = dtype == "c128"
    esz = 16 if c128 else 8
    ngroups = 0
    for po in offs:
        P = BE._at(blob, BE.Pass, po)
        if P.kind != 1 or not P.grouped:
            continue
        for gi in range(P.nops):
            g = BE._at(blob, BE.Group, po + P.ops_off + 256 * gi)
            ngroups += 1
            assert g.nvb == P.S - 4
            assert bool(g.pair16) == (not c128 and g.tpos[0] == 0)

            def raw_index(v, l):
                i = 0
                for b in range(g.nvb):
                    if (v >> b) & 1:
                        i |= g.vbit[b][0]
                for k in range(4):
                    if (l >> k) & 1:
                        i |= 1 << g.tpos[k]
                return i

            def addr(v, l):
                s = 0
                for b in range(g.nvb):
                    if (v >> b) & 1:
                        s ^= g.vbit[b][1]
                return s ^ g.sw_off[l]

            # precomputed per-thread bases (first 8 vector bits) agree with the bit table
            vt = np.frombuffer(blob, dtype=np.uint32, count=256, offset=po + g.vtab_off)
            for t in range(1 << min(g.nvb, 8)):
                raw = sum(g.vbit[b][0] for b in range(min(g.nvb, 8)) if (t >> b) & 1)
                sw = 0
                for b in range(min(g.nvb, 8)):
                    if (t >> b) & 1:
                        sw ^= g.vbit[b][1]
                assert int(vt[t]) == (sw & 0xFFFF) | (raw << 16)
            seen = set()
            for v in range(1 << g.nvb):
                for l in range(16):
                    i, a = raw_index(v, l), addr(v, l)
                    ci = i >> (0 if c128 else 1)
                    exp = _swz_slot(ci, P.swz_tma) if c128 else (_swz_slot(ci, P.swz_tma) << 1) | (i & 1)
                    assert a == exp
                    seen.add(a)
            assert len(seen) == 1 << P.S
            # bank-conflict freedom of one access instruction (fixed l, lanes vary v)
            vec16 = c128 or g.pair16
            lanes = 8 if vec16 else 16
            # banks reachable at all by the vector bits (small tiles may not span)
            reach = {((addr(v, 0) * esz) // (16 if vec16 else 8)) % (8 if vec16 else 16)
                     for v in range(1 << g.nvb)}
            want = min(lanes, len(reach))
            for l in (range(0, 16, 2) if (g.pair16 and not c128) else range(16)):
                for v0 in range(0, min(1 << g.nvb, 256), lanes):
                    banks = set()
                    for v in range(v0, min(v0 + lanes, 1 << g.nvb)):
                        byte = addr(v, l) * esz
                        banks.add((byte // (16 if vec16 else 8)) % (8 if vec16 else 16))
                    assert len(banks) == min(want, v0 + lanes if v0 + lanes <= (1 << g.nvb) else (1 << g.nvb) - v0), \
                        (case, gi, l, v0)
    assert ngroups > 0


@pytest.mark.parametrize("seed", range(12))
def test_flips_never_split_a_16B_pair(seed):
    """Predicated X flips folded into gather/scatter addresses (pass_format.h StvGroup.flip) must
    keep 16-B pair accesses aligned: a complex64 group that reads amplitude pairs never carries a
    flip of tile position 0; and the emulated blob still reproduces the oracle."""
    circ = C.qft_circuit(12, tail=200, seed=seed) if seed % 2 else \
        C.random_circuit(12, 250, seed, kinds=["cnot", "h", "cphase", "x", "cz", "t"])
    blob, offs = stv.plan_blob(circ.n, circ.gates)
    for po in offs:
        P = BE._at(blob, BE.Pass, po)
        if P.kind != 1 or not P.grouped:
            continue
        for i in range(P.nops):
            g = BE._at(blob, BE.Group, po + P.ops_off + 256 * i)
            fl = [g.flip[q] for q in range(g.nflip_g)] + [g.flip[8 + q] for q in range(g.nflip_s)]
            assert not (g.pair16 and any(f & 1 for f in fl))
    plan = stv.plan_json(circ.n, circ.gates)
    psi = PI.logical(plan, BE.run(circ.n, blob, offs, x0=circ.x0))
    assert np.max(np.abs(psi - oracle.run(circ))) < 2e-6


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("tile_bits", [0, 13])
def test_flip_targets_are_register_bits(seed, tile_bits):
    """Every predicated X flip folded into a group's gather or scatter addresses targets one of
    that group's 4 register bits (tpos): a flip of a vector bit would make the thread owning
    vector v read or write vector v^t's slots, and the group pass has no barrier between gather
    and scatter.  Covers flip-only groups merged into the previous group's scatter."""
    circ = C.random_circuit(22, 400, seed, kinds=["cnot", "x", "h", "cz", "t", "sx"])
    blob, offs = stv.plan_blob(circ.n, circ.gates, tile_bits=tile_bits)
    seen = 0
    for po in offs:
        P = BE._at(blob, BE.Pass, po)
        if P.kind != 1 or not P.grouped:
            continue
        for i in range(P.nops):
            g = BE._at(blob, BE.Group, po + P.ops_off + 256 * i)
            regs = {g.sw_off[1 << j] for j in range(4)}
            fl = [g.flip[q] for q in range(g.nflip_g)] + [g.flip[8 + q] for q in range(g.nflip_s)]
            seen += len(fl)
            assert all((f & 0xFFFF) in regs for f in fl), (po, i)
    assert seen > 0


@pytest.mark.parametrize("case", ["grid20", "c2", "c4", "rand"])
def test_tc_step_plan_structure(case):
    """Tensor-core step plans (pass_format.h StvTcStep): per group the steps cover its sub-op
    program in order without gaps; M steps hold only sub-ops that act the same on every
    vector of a tile (no V-bit tables, no V-bit-controlled CNOTs) and own distinct operator
    slots; the dependency masks contain every per-tile selector bit; tperm permutes the tile
    ordinal bits with the dependency bits on top."""
    # (tensor-core steps need full 12-bit tiles: c1's n = 16 plans 8-bit tiles on the CUDA-core
    # pass, so its 4x4-grid shape is taken at 4x5 = 20 qubits here)
    if case == "rand":
        circ = C.random_circuit(20, 400, 11)
    elif case == "grid20":
        circ = C.grid_circuit("g", 4, 5, 0, 20, "cz", 1)
    else:
        circ = C.config(int(case[1:]))
    blob, offs = stv.plan_blob(circ.n, circ.gates)
    npass = 0
    for po in offs:
        P = BE._at(blob, BE.Pass, po)
        if P.kind != 1 or not P.grouped or P.ntc == 0:
            continue
        npass += 1
        steps = [BE._at(blob, BE.TcStep, po + P.tc_off + 32 * i) for i in range(P.ntc)]
        groups = [BE._at(blob, BE.Group, po + P.ops_off + 256 * i) for i in range(P.nops)]
        out_bits = [b for b in range(64) if (P.out_mask >> b) & 1]
        ops = set()
        gi, pos = 0, 0
        for s in steps:
            assert s.group == gi and s.first == pos
            g = groups[gi]
            subs = [BE._at(blob, BE.Sub, po + g.sub_off + 16 * (s.first + k)) for k in range(s.n)]
            if s.kind == 1:
                slots = [s.op, s.op + 1] if s.bvar else [s.op]     # block variants: one slot per block
                assert not (set(slots) & ops) and max(slots) < P.ntcop
                ops.update(slots)
                bv = g.vbit[7][0] if g.nvb >= 8 else 0                # the block = vector bit 7
                uses_block = False
                for sb in subs:
                    c = sb.code & 0xFF
                    if 10 <= c < 30 and sb.ctl & 0xFFFF:                # V-bit control: only the block bit
                        assert sb.ctl & 0xFFFF == bv
                        uses_block = True
                    if c == 30 or 37 <= c < 41:
                        d = BE._at(blob, BE.DTab, po + P.tab_off + 48 * sb.arg)
                        assert d.m == 0 or (d.m == 1 and d.vraw[0] == bv)
                        uses_block |= d.m == 1
                    if 31 <= c < 37:
                        for i in range(3):
                            sel = (sb.code >> (8 + 5 * i)) & 31
                            if sel != 31:
                                assert (s.dep >> out_bits[sel]) & 1
                assert uses_block == bool(s.bvar)
            pos += s.n
            if s.last:
                assert pos == g.nsub
                gi, pos = gi + 1, 0
        assert gi == P.nops and len(ops) == P.ntcop
        nord = len(out_bits)
        perm = list(P.tperm)[:nord]
        assert sorted(perm) == list(range(nord))
        dep = 0
        for s in steps:
            if s.kind == 1:
                dep |= s.dep
        dep_ord = [i for i, b in enumerate(out_bits) if (dep >> b) & 1]
        assert sorted(perm[nord - len(dep_ord):]) == dep_ord
    assert npass > 0


@pytest.mark.parametrize("case", ["qft20", "rand20"])
def test_auto_low_run_full_tile_blob_semantics(case):
    """Full 12-bit tiles at n = 20: the tensor-core step encoding, tile-base terms sunk to the
    end of groups, and plan_auto's choice of the tile's low run L in {4, 5}: the automatic plan
    is the explicit plan of the L it chose, and both that plan and the explicit plan of the
    other L -- exact device blobs, emulated on CPU -- reproduce the oracle (complex64 bar 2e-6)."""
    circ = C.qft_circuit(20, tail=100, seed=3) if case == "qft20" else C.random_circuit(20, 300, 3)
    blob, offs = stv.plan_blob(circ.n, circ.gates)
    L0 = BE._at(blob, BE.Pass, offs[0]).L
    assert L0 in (4, 5)
    assert any(BE._at(blob, BE.Pass, po).ntc for po in offs)
    same, _ = stv.plan_blob(circ.n, circ.gates, low_bits=L0)
    assert bytes(same) == bytes(blob)
    other, offs_o = stv.plan_blob(circ.n, circ.gates, low_bits=9 - L0)   # explicit: no automatic choice
    assert bytes(other) != bytes(blob)
    ref = oracle.run(circ)
    for bl, of, lb in ((blob, offs, None), (other, offs_o, 9 - L0)):
        plan = stv.plan_json(circ.n, circ.gates, **({} if lb is None else dict(low_bits=lb)))
        psi = PI.logical(plan, BE.run(circ.n, bl, of, x0=circ.x0, c128=False))
        assert np.max(np.abs(psi - ref)) < 2e-6


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_vector_tables_and_half_local_boundaries(cfg):
    """Full-tile complex64 plans of c2-c4: every group's per-thread vector table equals the
    bases its vector bits define (the encoder re-chooses vector bit 7 after the groups are
    built), and at every boundary the tensor-core pass separates with a per-half barrier
    (same tile position at vector bit 7, no folded X flip across it; the kernel's hsync rule)
    thread t's half t >> 7 scatters in group o exactly the amplitudes it gathers in group o+1."""
    import struct
    c = C.config(cfg)
    blob, offs = stv.plan_blob(c.n, c.gates)
    nhalf = 0
    for po in offs:
        P = BE._at(blob, BE.Pass, po)
        if P.kind != 1 or not P.grouped or P.S != 12:
            continue
        gs = [BE._at(blob, BE.Group, po + P.ops_off + 256 * i) for i in range(P.nops)]
        halves = []
        for g in gs:
            sets = [set(), set()]
            for t in range(256):
                raw = sw = 0
                for v in range(8):
                    if (t >> v) & 1:
                        raw |= g.vbit[v][0]
                        sw ^= g.vbit[v][1]
                w = struct.unpack_from("<I", blob, po + g.vtab_off + 4 * t)[0]
                assert w == (sw & 0xFFFF) | (raw << 16)
                for l in range(16):
                    sets[t >> 7].add(raw | sum(1 << g.tpos[k] for k in range(4) if (l >> k) & 1))
            halves.append(sets)
        for o in range(len(gs) - 1):
            a, b = gs[o], gs[o + 1]
            s7 = a.vbit[7][1]
            ok = a.vbit[7][0] == b.vbit[7][0]
            ok = ok and all((a.flip[8 + q] & 0xFFFF) != s7 for q in range(a.nflip_s))
            ok = ok and all((b.flip[q] & 0xFFFF) != s7 for q in range(b.nflip_g))
            if ok:
                nhalf += 1
                assert halves[o][0] == halves[o + 1][0] and halves[o][1] == halves[o + 1][1]
    assert nhalf >= 3


def _tc_pass_launch_needs(n, gates, **kw):
    """(shared-memory bytes, kernel-parameter bytes, operator slots) of every tensor-core pass of a plan,
    as `launch_tc_group_pass` (kernels.cu) sizes them from the pass header."""
    blob, offs = stv.plan_blob(n, gates, **kw)
    out = []
    for po in offs:
        P = BE._at(blob, BE.Pass, po)
        if P.kind != 1 or not P.grouped or P.ntc == 0:
            continue
        smem = 2048 + P.ntcop * 8192 + 512 + ((P.tab_entries * 8 + 127) & ~127) + (8 << P.S)
        out.append((smem, P.param_bytes, P.ntcop))
    return out


@pytest.mark.parametrize("case", [("rand", 20, 43, dict(kmax=1)), ("rand", 20, 43, dict(kmax=2)),
                                  ("rand", 20, 43, dict(kmax=3)), ("rand", 20, 43, dict()),
                                  ("rand", 21, 12, dict(kmax=2)), ("rand", 22, 10, dict(kmax=3)),
                                  ("rand", 20, 7, dict(low_bits=5)), ("rand", 22, 5, dict(budget=400)),
                                  ("cfg", 2, 0, dict()), ("cfg", 2, 0, dict(kmax=2)), ("cfg", 2, 0, dict(kmax=3)),
                                  ("cfg", 3, 0, dict()), ("cfg", 4, 0, dict()), ("cfg", 4, 0, dict(kmax=3))])
def test_tc_passes_fit_the_launch_limits(case):
    """Every pass the encoder marks for the tensor-core kernel fits what its launch checks:
    113 KB of shared memory (one tile + operator slots + tables; 2 CTAs per SM), the 24 KB
    kernel-parameter part of the record and 12 operator slots.  (kmax = 2, 3 at n = 20 once encoded 10
    and 11 slots, 118 and 126 KB, and the launch failed with `invalid argument`.)"""
    kind, a, seed, kw = case
    c = C.random_circuit(a, 300, seed) if kind == "rand" else C.config(a)
    needs = _tc_pass_launch_needs(c.n, c.gates, **kw)
    assert needs, "no tensor-core pass in a full-tile complex64 plan"
    for smem, rec, slots in needs:
        assert smem <= 113 * 1024 and rec <= 24576 and 1 <= slots <= 12, (smem, rec, slots)
