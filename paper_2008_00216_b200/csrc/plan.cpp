// plan.cpp -- gate IR, relabel frame, Sec. 4.5 reordering, k-qubit fusion,
// diagonal clustering, global-qubit remap insertion, blob encoding.
// See plan.h for the step-by-step citations.
#include "plan.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <sstream>

namespace stv {

static const double kPi = 3.14159265358979323846;

// ---------------------------------------------------------------------------
// fixed-point turns
// ---------------------------------------------------------------------------
uint64_t turns_of_angle(double rad) {
    double x = rad / (2.0 * kPi);
    x -= std::nearbyint(x);               // [-0.5, 0.5]
    if (x >= 0.5) x -= 1.0;
    double y = std::ldexp(x, 64);         // |y| <= 2^63
    int64_t t = (y <= -9223372036854775808.0) ? INT64_MIN : (int64_t)std::llrint(y);
    return (uint64_t)t;
}

double angle_of_turns(uint64_t t) {
    return std::ldexp((double)(int64_t)t, -63) * kPi;
}

void QForm::add(const QForm &o) {
    cst += o.cst;
    for (auto &kv : o.lin) lin[kv.first] += kv.second;
    for (auto &kv : o.quad) quad[kv.first] += kv.second;
}

uint64_t QForm::eval(uint64_t j) const {
    uint64_t s = cst;
    for (auto &kv : lin)
        if ((j >> kv.first) & 1) s += kv.second;
    for (auto &kv : quad)
        if (((j >> kv.first.first) & 1) && ((j >> kv.first.second) & 1)) s += kv.second;
    return s;
}

uint64_t QForm::qubits() const {
    uint64_t m = 0;
    for (auto &kv : lin)
        if (kv.second) m |= 1ull << kv.first;
    for (auto &kv : quad)
        if (kv.second) m |= (1ull << kv.first.first) | (1ull << kv.first.second);
    return m;
}

bool QForm::trivial() const { return cst == 0 && qubits() == 0; }

uint64_t PGate::qmask() const {
    if (type == GType::DIAG) return form.qubits();
    uint64_t m = 0;
    for (int i = 0; i < nq; ++i) m |= 1ull << q[i];
    return m;
}

uint64_t PGate::dmask() const {
    if (type == GType::DIAG) return 0;
    if (type == GType::CNOT) return 1ull << q[1];
    return qmask();
}

void Frame::identity(int n) {
    for (int i = 0; i < 64; ++i) perm[i] = i;
    (void)n;
    xmask = 0;
}

// ---------------------------------------------------------------------------
// gate table (the product's own; written from PAPER.md L139-173 and the
// readings A3-A6 -- independent of oracle/)
// ---------------------------------------------------------------------------
static int nq_of(int kind) {
    switch (kind) {
    case SV_CZ: case SV_CNOT: case SV_SWAP: case SV_CPHASE: case SV_FSIM: case SV_U2: return 2;
    default: return 1;
    }
}

static void dense_matrix(const sv_gate &g, cd *U) {
    const double h = 0.70710678118654752440;   // 1/sqrt 2
    const cd I(0, 1);
    for (int i = 0; i < 16; ++i) U[i] = 0;
    switch (g.kind) {
    case SV_H: U[0] = h; U[1] = h; U[2] = h; U[3] = -h; break;
    case SV_X: U[1] = 1; U[2] = 1; break;
    case SV_Y: U[1] = -I; U[2] = I; break;
    case SV_Z: U[0] = 1; U[3] = -1; break;
    case SV_S: U[0] = 1; U[3] = I; break;
    case SV_T: U[0] = 1; U[3] = cd(h, h); break;
    case SV_SX: U[0] = cd(.5, .5); U[1] = cd(.5, -.5); U[2] = cd(.5, -.5); U[3] = cd(.5, .5); break;
    case SV_SY: U[0] = cd(.5, .5); U[1] = cd(.5, .5); U[2] = cd(-.5, -.5); U[3] = cd(.5, .5); break;
    case SV_SW: U[0] = cd(.5, .5); U[1] = cd(0, -h); U[2] = h; U[3] = cd(.5, .5); break;
    case SV_CZ: U[0] = 1; U[5] = 1; U[10] = 1; U[15] = -1; break;
    case SV_CNOT: U[0] = 1; U[5] = 1; U[11] = 1; U[14] = 1; break;
    case SV_SWAP: U[0] = 1; U[6] = 1; U[9] = 1; U[15] = 1; break;
    case SV_CPHASE: U[0] = 1; U[5] = 1; U[10] = 1; U[15] = std::polar(1.0, g.phi); break;
    case SV_FSIM:
        U[0] = 1; U[5] = std::cos(g.theta); U[6] = -I * std::sin(g.theta);
        U[9] = -I * std::sin(g.theta); U[10] = std::cos(g.theta); U[15] = std::polar(1.0, -g.phi);
        break;
    case SV_U1: for (int i = 0; i < 4; ++i) U[i] = cd(g.m[2 * i], g.m[2 * i + 1]); break;
    case SV_U2: for (int i = 0; i < 16; ++i) U[i] = cd(g.m[2 * i], g.m[2 * i + 1]); break;
    }
    if (g.flags & SV_GATE_ADJOINT) {
        int d = 1 << nq_of(g.kind);
        cd T[16];
        for (int r = 0; r < d; ++r)
            for (int c = 0; c < d; ++c) T[r * d + c] = std::conj(U[c * d + r]);
        std::memcpy((void *)U, (void *)T, sizeof(cd) * 16);
    }
}

std::string validate(int n, const sv_gate *g, size_t ng) {
    for (size_t i = 0; i < ng; ++i) {
        std::ostringstream e;
        const sv_gate &x = g[i];
        if (x.kind < 0 || x.kind >= SV_NUM_KINDS) { e << "gate " << i << ": unknown kind " << x.kind; return e.str(); }
        if (x.flags & ~SV_GATE_ADJOINT) { e << "gate " << i << ": unknown flags"; return e.str(); }
        int q = nq_of(x.kind);
        if (x.q0 < 0 || x.q0 >= n) { e << "gate " << i << ": qubit q0=" << x.q0 << " out of range [0," << n << ")"; return e.str(); }
        if (q == 2) {
            if (x.q1 < 0 || x.q1 >= n) { e << "gate " << i << ": qubit q1=" << x.q1 << " out of range"; return e.str(); }
            if (x.q1 == x.q0) { e << "gate " << i << ": duplicate qubit " << x.q0; return e.str(); }
        }
        if (!std::isfinite(x.theta) || !std::isfinite(x.phi)) { e << "gate " << i << ": non-finite angle"; return e.str(); }
        if (x.kind == SV_U1 || x.kind == SV_U2) {
            if (!x.m) { e << "gate " << i << ": NULL matrix"; return e.str(); }
            int d = 1 << q;
            for (int k = 0; k < 2 * d * d; ++k)
                if (!std::isfinite(x.m[k])) { e << "gate " << i << ": non-finite matrix entry"; return e.str(); }
            cd U[16];
            dense_matrix(x, U);
            double worst = 0;
            for (int r = 0; r < d; ++r)
                for (int c = 0; c < d; ++c) {
                    cd s = 0;
                    for (int k = 0; k < d; ++k) s += std::conj(U[k * d + r]) * U[k * d + c];
                    worst = std::max(worst, std::abs(s - cd(r == c ? 1.0 : 0.0)));
                }
            if (worst > 1e-10) { e << "gate " << i << ": matrix not unitary (|U^dag U - I| = " << worst << ")"; return e.str(); }
        }
    }
    return "";
}

// ---------------------------------------------------------------------------
// a1 + a2: classification and the relabel frame
// ---------------------------------------------------------------------------
// diagonal table t[l] (l = local index, q[0] = MSB) -> QForm over bits p[]
static QForm form_of_table(int nq, const int *p, const uint64_t *t) {
    QForm f;
    if (nq == 1) {
        f.cst = t[0];
        f.lin[p[0]] = t[1] - t[0];
    } else {
        // l = 2 b(p0) + b(p1)
        f.cst = t[0];
        f.lin[p[1]] = t[1] - t[0];
        f.lin[p[0]] = t[2] - t[0];
        int a = std::min(p[0], p[1]), b = std::max(p[0], p[1]);
        f.quad[{a, b}] = t[3] - t[2] - t[1] + t[0];
    }
    for (auto it = f.lin.begin(); it != f.lin.end();) it = it->second ? std::next(it) : f.lin.erase(it);
    for (auto it = f.quad.begin(); it != f.quad.end();) it = it->second ? std::next(it) : f.quad.erase(it);
    return f;
}

static bool is_diag(int d, const cd *U) {
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c)
            if (r != c && U[r * d + c] != cd(0, 0)) return false;
    return true;
}

std::vector<PGate> to_physical(int n, const sv_gate *gs, size_t ng, Frame &fr, uint32_t flags) {
    (void)n;
    std::vector<PGate> out;
    out.reserve(ng);
    const bool relabel = !(flags & SV_OPT_NO_RELABEL);
    const uint64_t Q = 1ull << 62, H = 1ull << 63, E = 1ull << 61;  // quarter, half, eighth turn
    for (size_t i = 0; i < ng; ++i) {
        const sv_gate &g = gs[i];
        const bool adj = g.flags & SV_GATE_ADJOINT;
        const int nq = nq_of(g.kind);
        int lq[2] = {g.q0, nq == 2 ? g.q1 : -1};
        int p[2] = {fr.perm[lq[0]], nq == 2 ? fr.perm[lq[1]] : -1};
        int f[2] = {(int)((fr.xmask >> p[0]) & 1), nq == 2 ? (int)((fr.xmask >> p[1]) & 1) : 0};
        const int F = nq == 2 ? (f[0] << 1) | f[1] : f[0];
        auto emit_diag = [&](const uint64_t *tlog) {
            uint64_t t[4];
            for (int l = 0; l < (1 << nq); ++l) t[l ^ F] = adj ? (uint64_t)(0 - tlog[l]) : tlog[l];
            PGate pg;
            pg.type = GType::DIAG;
            pg.nq = nq;
            pg.q[0] = p[0]; pg.q[1] = p[1];
            pg.form = form_of_table(nq, p, t);
            pg.src = (int)i;
            if (!pg.form.trivial()) out.push_back(pg);
        };
        auto emit_dense = [&]() {
            cd U[16];
            dense_matrix(g, U);
            int d = 1 << nq;
            PGate pg;
            pg.type = GType::DENSE;
            pg.nq = nq;
            pg.q[0] = p[0]; pg.q[1] = p[1];
            for (int r = 0; r < d; ++r)
                for (int c = 0; c < d; ++c) pg.U[(r ^ F) * d + (c ^ F)] = U[r * d + c];
            pg.src = (int)i;
            if (is_diag(d, pg.U)) {       // e.g. Eq. 2-style products, diagonal U1/U2
                uint64_t t[4];
                for (int l = 0; l < d; ++l) t[l] = turns_of_angle(std::arg(pg.U[l * d + l]));
                PGate dg;
                dg.type = GType::DIAG;
                dg.nq = nq;
                dg.q[0] = p[0]; dg.q[1] = p[1];
                dg.form = form_of_table(nq, p, t);
                dg.src = (int)i;
                if (!dg.form.trivial()) out.push_back(dg);
                return;
            }
            out.push_back(pg);
        };
        switch (g.kind) {
        case SV_Z: { uint64_t t[2] = {0, H}; emit_diag(t); break; }
        case SV_S: { uint64_t t[2] = {0, Q}; emit_diag(t); break; }
        case SV_T: { uint64_t t[2] = {0, E}; emit_diag(t); break; }
        case SV_CZ: { uint64_t t[4] = {0, 0, 0, H}; emit_diag(t); break; }
        case SV_CPHASE: { uint64_t t[4] = {0, 0, 0, turns_of_angle(g.phi)}; emit_diag(t); break; }
        case SV_X:
            if (relabel) fr.xmask ^= 1ull << p[0]; else emit_dense();
            break;
        case SV_Y:
            if (relabel) {
                // Y = X . diag(i, -i): apply the diagonal, then relabel X.
                // Y is self-inverse: pre-negate so emit_diag's adjoint negation cancels
                uint64_t t[2] = {adj ? 3 * Q : Q, adj ? Q : 3 * Q};
                emit_diag(t);
                fr.xmask ^= 1ull << p[0];
            } else emit_dense();
            break;
        case SV_SWAP:
            if (relabel) std::swap(fr.perm[lq[0]], fr.perm[lq[1]]); else emit_dense();
            break;
        case SV_CNOT: {
            PGate pg;
            pg.type = GType::CNOT;
            pg.nq = 2;
            pg.q[0] = p[0]; pg.q[1] = p[1];
            pg.src = (int)i;
            out.push_back(pg);
            // a flipped control turns CNOT into X_t . CNOT: relabel the X
            if (f[0]) fr.xmask ^= 1ull << p[1];
            break;
        }
        case SV_FSIM:
            if (relabel && g.theta == kPi / 2) {
                // reading A5: fSim(pi/2, phi) = SWAP . diag(1, -i, -i, e^{-i phi})
                uint64_t t[4] = {0, 3 * Q, 3 * Q, turns_of_angle(-g.phi)};
                emit_diag(t);
                std::swap(fr.perm[lq[0]], fr.perm[lq[1]]);
            } else emit_dense();
            break;
        case SV_U1:
            if (relabel) {
                cd U[16];
                dense_matrix(g, U);
                if (U[0] == cd(0, 0) && U[3] == cd(0, 0)) {
                    // anti-diagonal [[0,b],[a,0]] = X . diag(a, b)
                    uint64_t t[2] = {turns_of_angle(std::arg(U[2])), turns_of_angle(std::arg(U[1]))};
                    const bool a0 = adj;
                    (void)a0;
                    // dense_matrix already applied the adjoint; emit_diag must not negate again
                    PGate pg;
                    uint64_t tt[2];
                    for (int l = 0; l < 2; ++l) tt[l ^ F] = t[l];
                    pg.type = GType::DIAG;
                    pg.nq = 1;
                    pg.q[0] = p[0];
                    pg.form = form_of_table(1, p, tt);
                    pg.src = (int)i;
                    if (!pg.form.trivial()) out.push_back(pg);
                    fr.xmask ^= 1ull << p[0];
                    break;
                }
            }
            emit_dense();
            break;
        default:
            emit_dense();
        }
    }
    return out;
}

// ---------------------------------------------------------------------------
// dense-matrix helpers (local index LSB-first over an ascending bit list)
// ---------------------------------------------------------------------------
// Expand gate matrix G (nq qubits, q[0] = MSB) to the basis of ascending bits tg.
static std::vector<cd> expand_gate(const PGate &g, const std::vector<int> &tg) {
    const int k = (int)tg.size(), D = 1 << k;
    int pos[2];
    for (int i = 0; i < g.nq; ++i) pos[i] = (int)(std::find(tg.begin(), tg.end(), g.q[i]) - tg.begin());
    uint32_t gm = 0;
    for (int i = 0; i < g.nq; ++i) gm |= 1u << pos[i];
    const int d = 1 << g.nq;
    std::vector<cd> R((size_t)D * D, cd(0, 0));
    for (int r = 0; r < D; ++r)
        for (int c = 0; c < D; ++c) {
            if ((r & ~gm) != (c & ~gm)) continue;
            int lr = 0, lc = 0;
            for (int i = 0; i < g.nq; ++i) {
                lr |= ((r >> pos[i]) & 1) << (g.nq - 1 - i);
                lc |= ((c >> pos[i]) & 1) << (g.nq - 1 - i);
            }
            R[(size_t)r * D + c] = g.U[lr * d + lc];
        }
    return R;
}

// Re-express op matrix M over `from` bits in the basis of `to` (superset) bits.
static std::vector<cd> widen(const std::vector<cd> &M, const std::vector<int> &from, const std::vector<int> &to) {
    const int k = (int)to.size(), D = 1 << k, kf = (int)from.size(), Df = 1 << kf;
    std::vector<int> pos(kf);
    uint32_t fm = 0;
    for (int i = 0; i < kf; ++i) {
        pos[i] = (int)(std::find(to.begin(), to.end(), from[i]) - to.begin());
        fm |= 1u << pos[i];
    }
    std::vector<cd> R((size_t)D * D, cd(0, 0));
    for (int r = 0; r < D; ++r)
        for (int c = 0; c < D; ++c) {
            if ((r & ~fm) != (c & ~fm)) continue;
            int lr = 0, lc = 0;
            for (int i = 0; i < kf; ++i) {
                lr |= ((r >> pos[i]) & 1) << i;
                lc |= ((c >> pos[i]) & 1) << i;
            }
            R[(size_t)r * D + c] = M[(size_t)lr * Df + lc];
        }
    return R;
}

static std::vector<cd> matmul(const std::vector<cd> &A, const std::vector<cd> &B, int D) {
    std::vector<cd> C((size_t)D * D, cd(0, 0));
    for (int r = 0; r < D; ++r)
        for (int k = 0; k < D; ++k) {
            cd a = A[(size_t)r * D + k];
            if (a == cd(0, 0)) continue;
            for (int c = 0; c < D; ++c) C[(size_t)r * D + c] += a * B[(size_t)k * D + c];
        }
    return C;
}

static std::vector<int> bits_of(uint64_t m) {
    std::vector<int> v;
    for (int b = 0; b < 64; ++b)
        if ((m >> b) & 1) v.push_back(b);
    return v;
}

// ---------------------------------------------------------------------------
// a3 + a4: reordering + fusion into passes
// ---------------------------------------------------------------------------
PlanOptions resolve_options(const sv_options *o, int amp_bytes, int n_local) {
    PlanOptions p;
    p.tile_bits = amp_bytes == 8 ? 12 : 11;
    if (o) {
        if (o->kmax > 0) p.kmax = std::min(o->kmax, STV_MAX_K);
        if (o->tile_bits > 0) p.tile_bits = std::min(o->tile_bits, STV_MAX_TILE_BITS);
        if (o->low_bits > 0) { p.low_bits = o->low_bits; p.low_auto = false; }
        if (o->budget > 0) p.budget = o->budget;
        p.flags = o->flags;
    }
    // shared memory: 3 stages of 2^S amplitudes + matrices must fit in 227 KB
    p.tile_bits = std::min(p.tile_bits, amp_bytes == 8 ? 13 : 12);
    // keep >= ~256 tiles so every SM gets work; small states get small tiles
    int smax = std::min(p.tile_bits, std::max(std::min(n_local, 6), n_local - 8));
    p.tile_bits = std::max(1, std::min(smax, n_local));
    // TMA bulk copies move >= 16 B: c64 runs need >= 2 amplitudes (L >= 1)
    const int minL = amp_bytes == 8 ? 1 : 0;
    p.low_bits = std::max(minL, std::min(p.low_bits, p.tile_bits - 2));
    p.tile_bits = std::max(p.tile_bits, std::min(n_local, p.low_bits + 2));   // any 2-qubit gate fits
    p.kmax = std::max(1, std::min(p.kmax, p.tile_bits));
    return p;
}

static const size_t kMaxRecBytes = 24576;   // pass record (ops, matrices, diag forms) staged in smem

// Per-amplitude instruction estimate of one op on a resident tile (thread
// instructions: FMAs, shared-memory traffic, addressing); calibrated against
// the ncu instruction counts of k_tile_pass (profiles/).
static int op_cost(const FOp &o) {
    switch (o.type) {
    case OP_DENSE: {
        static const int c[5] = {0, 12, 22, 44, 84};
        return c[std::min<size_t>(o.tg.size(), 4)];
    }
    case OP_DIAG: return 30;
    default: return 6;
    }
}

static bool commutes_op(const FOp &o, uint64_t gq, uint64_t gd) {
    // commute iff on every shared qubit both act diagonally
    uint64_t shared = o.qmask & gq;
    return (shared & (o.dmask | gd)) == 0;
}

// Try to merge gate g (actual-physical bits) into the op list (backward search).
static void merge_into(std::vector<FOp> &ops, const PGate &g, int kmax, bool fold_diag, bool one_gate) {
    const uint64_t gq = g.qmask(), gd = g.dmask();
    if (!one_gate) {
        for (int i = (int)ops.size() - 1; i >= 0; --i) {
            FOp &o = ops[i];
            bool ok = false;
            if (g.type == GType::DIAG) {
                if (o.type == OP_DIAG) ok = true;
                else if (o.type == OP_DENSE && fold_diag && (gq & ~o.dmask) == 0) ok = true;
            } else if (g.type == GType::DENSE && o.type == OP_DENSE) {
                ok = __builtin_popcountll(o.dmask | gd) <= kmax;
            } else if (g.type == GType::CNOT && o.type == OP_DENSE) {
                ok = (gq & ~o.dmask) == 0;    // CNOT inside the op's targets: a 4x4 permutation factor
            }
            if (ok) {
                if (g.type == GType::DIAG && o.type == OP_DIAG) {
                    o.form.add(g.form);
                    o.qmask |= gq;
                } else {
                    uint64_t nm = o.dmask | gq;
                    std::vector<int> tg = bits_of(nm);
                    std::vector<cd> Mw = widen(o.M, o.tg, tg);
                    std::vector<cd> G;
                    if (g.type == GType::DIAG) {
                        const int D = 1 << (int)tg.size();
                        G.assign((size_t)D * D, cd(0, 0));
                        for (int l = 0; l < D; ++l) {
                            uint64_t j = 0;
                            for (size_t b = 0; b < tg.size(); ++b)
                                if ((l >> b) & 1) j |= 1ull << tg[b];
                            G[(size_t)l * D + l] = std::polar(1.0, angle_of_turns(g.form.eval(j)));
                        }
                    } else if (g.type == GType::CNOT) {
                        PGate pc = g;
                        for (int r = 0; r < 16; ++r) pc.U[r] = 0;
                        pc.U[0] = 1; pc.U[5] = 1; pc.U[11] = 1; pc.U[14] = 1;
                        G = expand_gate(pc, tg);
                    } else {
                        G = expand_gate(g, tg);
                    }
                    o.M = matmul(G, Mw, 1 << (int)tg.size());
                    o.tg = tg;
                    o.qmask = o.dmask = nm;
                }
                return;
            }
            if (!commutes_op(o, gq, gd)) break;
        }
    }
    FOp o;
    if (g.type == GType::DIAG) {
        o.type = OP_DIAG;
        o.form = g.form;
        o.qmask = gq;
        o.dmask = 0;
    } else if (g.type == GType::CNOT) {
        o.type = OP_CNOT;
        o.c = g.q[0];
        o.t = g.q[1];
        o.qmask = gq;
        o.dmask = gd;
    } else {
        o.type = OP_DENSE;
        o.tg = bits_of(gq);
        o.M = expand_gate(g, o.tg);
        o.qmask = o.dmask = gq;
    }
    ops.push_back(o);
}

static PGate map_gate(const PGate &g, const int *sigma) {
    PGate a = g;
    for (int i = 0; i < g.nq; ++i) a.q[i] = sigma[g.q[i]];
    if (g.type == GType::DIAG) {
        QForm f;
        f.cst = g.form.cst;
        for (auto &kv : g.form.lin) f.lin[sigma[kv.first]] += kv.second;
        for (auto &kv : g.form.quad) {
            int x = sigma[kv.first.first], y = sigma[kv.first.second];
            f.quad[{std::min(x, y), std::max(x, y)}] += kv.second;
        }
        a.form = f;
    }
    return a;
}

// ---------------------------------------------------------------------------
// register-resident gate groups (OP_GROUP): the pass's gates are partitioned
// into groups whose in-tile qubits fit in STV_GROUP_BITS tile bits; a group is
// one shared-memory round trip of the tile, its gates run as sub-ops on
// 16-amplitude register vectors (the paper's "clusters
// stored in factored form").  The partition is the Sec. 4.5 scan
// again at op level: a gate joins the open group iff it commutes with every
// gate skipped so far and its in-tile qubits still fit.
// ---------------------------------------------------------------------------
static int sub_cost(const FOp &o) {
    switch (o.type) {
    case OP_DENSE: return o.tg.size() == 1 ? 10 : 20;
    case OP_DIAG: return 6;
    default: return 2;
    }
}

struct GroupScan {              // final state of one group's scan (for incremental adds)
    uint64_t T = 0, blockedAll = 0, blockedDense = 0;
};

struct OpsEval {
    std::vector<FOp> ops;
    std::vector<GroupScan> scan;  // parallel to ops in group mode
    bool grouped = false;
    int cost = 0;
    size_t rec = 0;
    size_t tab = 0;           // shared-memory bytes of the group diag tables
    int ntab = 0;
};

// Shared-memory bytes (pass record + table area) of a group diagonal sub-op:
// the greedy split of its terms into tables of <= STV_MAX_VBITS V-bits
// (vmask = in-tile qubits outside the group; mirrors split_group_diag).
static size_t diag_table_bytes(const QForm &f, uint64_t vmask, uint64_t T, int amp_bytes, int *ntab,
                               size_t *tab_smem) {
    // one half table when every term contains one group bit j (mirrors half_table)
    if (f.cst == 0)
        for (uint64_t tt = T; tt; tt &= tt - 1) {
            const int j = __builtin_ctzll(tt);
            bool ok = true;
            uint64_t vb = 0;
            for (auto &kv : f.lin) ok &= kv.first == j;
            for (auto &kv : f.quad) {
                const int x = kv.first.first, y = kv.first.second;
                if (x != j && y != j) { ok = false; break; }
                vb |= vmask & (1ull << (x == j ? y : x));
            }
            const int m = __builtin_popcountll(vb);
            if (!ok || m > STV_MAX_VBITS_H) continue;
            *ntab = 1;
            *tab_smem += (size_t)(STV_TAB_STRIDE_H * amp_bytes) << m;
            return sizeof(StvDTab) + sizeof(StvSub) + 32 + sizeof(StvTerm) * (f.lin.size() + f.quad.size());
        }
    std::vector<uint64_t> sets;
    auto place = [&](uint64_t need) {
        for (uint64_t &u : sets)
            if (__builtin_popcountll(u | need) <= STV_MAX_VBITS) { u |= need; return; }
        sets.push_back(need);
    };
    size_t terms = 0;
    for (auto &kv : f.lin) place(vmask & (1ull << kv.first));
    for (auto &kv : f.quad) place(vmask & ((1ull << kv.first.first) | (1ull << kv.first.second)));
    terms = f.lin.size() + f.quad.size();
    if (sets.empty()) sets.push_back(0);
    size_t bytes = sizeof(StvTerm) * terms;
    for (uint64_t u : sets) {
        const int m = __builtin_popcountll(u);
        bytes += sizeof(StvDTab) + sizeof(StvSub) + 32;
        *tab_smem += (size_t)(STV_TAB_STRIDE * amp_bytes) << m;
    }
    *ntab = (int)sets.size();
    return bytes;
}

static void tally(OpsEval &ev, int amp_bytes, uint64_t S = 0) {
    ev.cost = 0;
    ev.rec = sizeof(StvPass);
    ev.tab = 0;
    ev.ntab = 0;
    for (auto &grp : ev.ops) {
        if (grp.type != OP_GROUP) {
            ev.cost += op_cost(grp);
            ev.rec += sizeof(StvOp);
            if (grp.type == OP_DENSE) ev.rec += (size_t)amp_bytes << (2 * grp.tg.size());
            if (grp.type == OP_DIAG)
                ev.rec += sizeof(StvDiag) + sizeof(StvTerm) * (grp.form.lin.size() + grp.form.quad.size());
            continue;
        }
        for (auto &o : grp.subs) {
            ev.cost += sub_cost(o);
            ev.rec += sizeof(StvSub);
            if (o.type == OP_DENSE) ev.rec += (size_t)amp_bytes << (2 * o.tg.size());
            if (o.type == OP_DIAG) {
                // per-tile tables over the group bits + V-bits, split as the encoder does
                int ntb = 0;
                ev.rec += diag_table_bytes(o.form, S & ~grp.T, grp.T, amp_bytes, &ntb, &ev.tab);
                ev.ntab += ntb;
            }
        }
        ev.cost += 16;                           // the group's shared-memory round trip
        ev.rec += sizeof(StvGroup);
    }
}

static OpsEval make_ops(const std::vector<PGate> &gs, uint64_t S, const PlanOptions &opt, int amp_bytes) {
    OpsEval ev;
    const bool fold = !(opt.flags & SV_OPT_NO_DIAG_FOLD);
    const bool one_gate = opt.flags & SV_OPT_ONE_GATE;
    if ((opt.flags & SV_OPT_NO_GROUPS) || one_gate || opt.tile_bits < STV_GROUP_BITS) {
        for (const PGate &g : gs) merge_into(ev.ops, g, opt.kmax, fold, one_gate);
        tally(ev, amp_bytes);
        return ev;
    }
    ev.grouped = true;
    std::vector<char> taken(gs.size(), 0);
    size_t first = 0;
    while (true) {
        while (first < gs.size() && taken[first]) ++first;
        if (first >= gs.size()) break;
        FOp grp;
        grp.type = OP_GROUP;
        GroupScan sc;
        for (size_t i = first; i < gs.size(); ++i) {
            if (taken[i]) continue;
            const PGate &g = gs[i];
            const uint64_t qm = g.qmask(), dm = g.dmask();
            // diagonal gates never claim register bits: their in-tile qubits outside
            // the group become per-vector terms ("V-bits")
            const uint64_t in_tile = (g.type == GType::DIAG ? 0 : dm) & S;
            // kmax bounds the register bits (the dense block size) of a group: <= 4 (16-amplitude
            // vectors); a gate wider than kmax still gets a group of its own
            const int lim = std::max(std::min(opt.kmax, STV_GROUP_BITS), __builtin_popcountll(in_tile));
            bool ok = !(qm & sc.blockedAll) && !(dm & sc.blockedDense) && __builtin_popcountll(sc.T | in_tile) <= lim;
            if (!ok) {
                sc.blockedAll |= dm;
                sc.blockedDense |= qm & ~dm;
                continue;
            }
            merge_into(grp.subs, g, 2, fold, false);
            sc.T |= in_tile;
            taken[i] = 1;
        }
        grp.T = sc.T;
        for (auto &o : grp.subs) {
            grp.qmask |= o.qmask;
            grp.dmask |= o.dmask;
        }
        ev.ops.push_back(std::move(grp));
        ev.scan.push_back(sc);
    }
    tally(ev, amp_bytes, S);
    return ev;
}

// Add gate g (last in scan order) to an existing group partition: exactly what
// make_ops would decide, since earlier decisions never depend on later gates
// (valid while the tile set S is unchanged).
static void add_gate(OpsEval &ev, const PGate &g, uint64_t S, const PlanOptions &opt, int amp_bytes) {
    const bool fold = !(opt.flags & SV_OPT_NO_DIAG_FOLD);
    const uint64_t qm = g.qmask(), dm = g.dmask();
    const uint64_t in_tile = (g.type == GType::DIAG ? 0 : dm) & S;
    bool placed = false;
    for (size_t k = 0; k < ev.ops.size() && !placed; ++k) {
        GroupScan &sc = ev.scan[k];
        bool ok = !(qm & sc.blockedAll) && !(dm & sc.blockedDense) &&
                  __builtin_popcountll(sc.T | in_tile) <= STV_GROUP_BITS;
        if (!ok) {
            sc.blockedAll |= dm;
            sc.blockedDense |= qm & ~dm;
            continue;
        }
        FOp &grp = ev.ops[k];
        merge_into(grp.subs, g, 2, fold, false);
        sc.T |= in_tile;
        grp.T = sc.T;
        grp.qmask |= qm;
        grp.dmask |= dm;
        placed = true;
    }
    if (!placed) {
        FOp grp;
        grp.type = OP_GROUP;
        GroupScan sc;
        merge_into(grp.subs, g, 2, fold, false);
        sc.T = in_tile;
        grp.T = sc.T;
        grp.qmask = qm;
        grp.dmask = dm;
        ev.ops.push_back(std::move(grp));
        ev.scan.push_back(sc);
    }
    // sub-op masks may have been merged: recompute the group masks exactly
    for (auto &grp : ev.ops) {
        grp.qmask = grp.dmask = 0;
        for (auto &o : grp.subs) {
            grp.qmask |= o.qmask;
            grp.dmask |= o.dmask;
        }
    }
    tally(ev, amp_bytes, S);
}

// ---------------------------------------------------------------------------
// Chains of 2-qubit sub-ops on the same pair P inside a gate group, separated
// only by ops on other bits and by diagonal sub-ops whose terms on P couple P
// to bits OUTSIDE the tile, are one 4x4 operator per tile: the diagonal factor
// on P is fixed once the tile's outside bits are.  The chain becomes one dense
// sub-op with 2^|sel| per-tile variants (products in complex128, rounded once;
// Eq. 2 coalescing of PAPER.md L645-653 with the phases of P:L503-527 bound
// per tile).  The kernel picks the variant from the tile base (a uniform
// index) -- the parts of the diagonals on other bits stay as they were.
// ---------------------------------------------------------------------------
static const int kMaxSel = 3;

static std::vector<cd> diag_on_pair(const QForm &part, int a, int b, const std::vector<int> &sel, int v) {
    // 4x4 diagonal over P = (a < b) (local index bit0 = a, bit1 = b) for selector assignment v
    std::vector<cd> D(16, cd(0, 0));
    for (int l = 0; l < 4; ++l) {
        uint64_t j = 0;
        if (l & 1) j |= 1ull << a;
        if (l & 2) j |= 1ull << b;
        for (size_t i = 0; i < sel.size(); ++i)
            if ((v >> i) & 1) j |= 1ull << sel[i];
        D[(size_t)l * 4 + l] = std::polar(1.0, angle_of_turns(part.eval(j)));
    }
    return D;
}

// Re-express dense op o (2 qubits, maybe with variants) over selector set `sel`
// and multiply the diagonal `part` (over o's pair + selector bits) on the left
// (after o) or on the right (before o).
static void fold_diag_into(FOp &o, const QForm &part, const std::vector<int> &part_sel, bool after) {
    std::vector<int> sel = o.sel;
    for (int x : part_sel)
        if (std::find(sel.begin(), sel.end(), x) == sel.end()) sel.push_back(x);
    std::sort(sel.begin(), sel.end());
    const int nv = 1 << (int)sel.size();
    const int a = o.tg[0], b = o.tg[1];
    std::vector<std::vector<cd>> Mv((size_t)nv);
    for (int v = 0; v < nv; ++v) {
        int w = 0;
        for (size_t q = 0; q < o.sel.size(); ++q) {
            const size_t pos = std::find(sel.begin(), sel.end(), o.sel[q]) - sel.begin();
            if ((v >> pos) & 1) w |= 1 << q;
        }
        const std::vector<cd> &M = o.Mv.empty() ? o.M : o.Mv[(size_t)w];
        const std::vector<cd> D = diag_on_pair(part, a, b, sel, v);
        Mv[(size_t)v] = after ? matmul(D, M, 4) : matmul(M, D, 4);
    }
    o.Mv = Mv;
    o.sel = sel;
    o.M = Mv[0];
}

// Move the parts of group diagonal sub-ops that a neighbouring 2-qubit dense
// sub-op can carry as per-tile variants into that op: for a group bit j, the
// terms of the diagonal on j (linear, and pairs with bits OUTSIDE the tile)
// commute with every op that acts on j only diagonally, so they slide to the
// previous or next dense op on j and become part of its matrix (the outside
// bits become selectors).  Constant and outside-only terms are per-tile
// scalars and ride on any dense op.  Terms on two in-tile bits stay.
// Pass level: a diagonal term none of whose bits is one of its group's register
// bits (a "V-bit" term) moves to the nearest group of the pass that holds one of
// its in-tile bits in registers, provided no group in between acts non-diagonally
// on its bits (diagonal terms commute with everything else).  There it is a
// group-bit term that absorb_diagonals can fold into a matrix, instead of a
// per-vector table factor.
static void relocate_v_terms(std::vector<FOp> &ops, uint64_t S) {
    const int ng = (int)ops.size();
    for (int a = 0; a < ng; ++a) {
        if (ops[a].type != OP_GROUP) continue;
        for (FOp &d : ops[a].subs) {
            if (d.type != OP_DIAG) continue;
            const uint64_t TA = ops[a].T;
            std::vector<std::pair<std::vector<int>, uint64_t>> moved_terms;   // (bits, angle) per target group
            auto try_move = [&](uint64_t X) -> int {
                if ((X & TA) || !(X & S)) return -1;                 // touches A's bits, or outside only
                int best = -1, bd = 1 << 30;
                for (int dir : {1, -1}) {
                    for (int b = a + dir; b >= 0 && b < ng; b += dir) {
                        if (ops[b].type != OP_GROUP) break;
                        if (ops[b].T & X & S) {                          // holds one of the bits: target
                            if (std::abs(b - a) < bd) { bd = std::abs(b - a); best = b; }
                            break;
                        }
                        if (ops[b].dmask & X) break;                     // blocked
                    }
                }
                return best;
            };
            std::vector<std::vector<QForm>> add(ng);
            for (auto it = d.form.lin.begin(); it != d.form.lin.end();) {
                const int b = try_move(1ull << it->first);
                if (b >= 0) {
                    QForm q;
                    q.lin[it->first] = it->second;
                    add[b].push_back(q);
                    it = d.form.lin.erase(it);
                } else ++it;
            }
            for (auto it = d.form.quad.begin(); it != d.form.quad.end();) {
                const int b = try_move((1ull << it->first.first) | (1ull << it->first.second));
                if (b >= 0) {
                    QForm q;
                    q.quad[it->first] = it->second;
                    add[b].push_back(q);
                    it = d.form.quad.erase(it);
                } else ++it;
            }
            d.qmask = d.form.qubits();
            for (int b = 0; b < ng; ++b) {
                if (add[b].empty()) continue;
                FOp nd;
                nd.type = OP_DIAG;
                for (const QForm &q : add[b]) nd.form.add(q);
                nd.qmask = nd.form.qubits();
                std::vector<FOp> &sb = ops[b].subs;
                if (b > a) sb.insert(sb.begin(), nd);                  // later group: at its start
                else sb.push_back(nd);                                  // earlier group: at its end
                ops[b].qmask |= nd.qmask;
            }
        }
        auto &sb = ops[a].subs;
        for (size_t k = 0; k < sb.size();) {
            if (sb[k].type == OP_DIAG && sb[k].form.trivial()) sb.erase(sb.begin() + (long)k);
            else ++k;
        }
    }
}

static void absorb_diagonals(FOp &grp, uint64_t S, int nl) {
    std::vector<FOp> &ops = grp.subs;
    const uint64_t sel_ok = ~0ull;   // global-bit selectors are resolved per rank at encode time
    (void)nl;
    auto is_pair_dense = [](const FOp &o) { return o.type == OP_DENSE && o.tg.size() == 2; };
    for (size_t k = 0; k < ops.size(); ++k) {
        if (ops[k].type != OP_DIAG) continue;
        QForm &F = ops[k].form;
        // candidate group bits: in-tile bits with movable terms
        std::vector<int> bits;
        for (auto &kv : F.lin)
            if ((S >> kv.first) & 1) bits.push_back(kv.first);
        for (auto &kv : F.quad) {
            const int x = kv.first.first, y = kv.first.second;
            const bool ix = (S >> x) & 1, iy = (S >> y) & 1;
            if (ix != iy) bits.push_back(ix ? x : y);
        }
        std::sort(bits.begin(), bits.end());
        bits.erase(std::unique(bits.begin(), bits.end()), bits.end());
        for (int j : bits) {
            QForm part;
            std::vector<int> psel;
            bool ok = true;
            if (F.lin.count(j)) part.lin[j] = F.lin[j];
            for (auto &kv : F.quad) {
                const int x = kv.first.first, y = kv.first.second;
                if (x != j && y != j) continue;
                const int other = x == j ? y : x;
                if ((S >> other) & 1) continue;                      // in-tile partner: stays
                if (!((sel_ok >> other) & 1)) { ok = false; break; }
                part.quad[kv.first] = kv.second;
                if (std::find(psel.begin(), psel.end(), other) == psel.end()) psel.push_back(other);
            }
            if (!ok || (part.lin.empty() && part.quad.empty())) continue;
            // nearest ops acting on j non-diagonally, before and after
            int prev = -1, next = -1;
            for (int i = (int)k - 1; i >= 0; --i)
                if ((ops[i].dmask >> j) & 1) { prev = i; break; }
            for (size_t i = k + 1; i < ops.size(); ++i)
                if ((ops[i].dmask >> j) & 1) { next = (int)i; break; }
            auto nsel_after = [&](int i) {
                std::vector<int> s2 = ops[i].sel;
                for (int x : psel)
                    if (std::find(s2.begin(), s2.end(), x) == s2.end()) s2.push_back(x);
                return (int)s2.size();
            };
            int tgt = -1;
            bool after = false;
            const int cn = next >= 0 && is_pair_dense(ops[next]) ? nsel_after(next) : 99;
            const int cp = prev >= 0 && is_pair_dense(ops[prev]) ? nsel_after(prev) : 99;
            if (cn <= kMaxSel && cn <= cp) { tgt = next; after = false; }
            else if (cp <= kMaxSel) { tgt = prev; after = true; }
            if (tgt < 0) continue;
            fold_diag_into(ops[tgt], part, psel, after);
            for (auto &kv : part.lin) F.lin.erase(kv.first);
            for (auto &kv : part.quad) F.quad.erase(kv.first);
        }
        // per-tile scalars: constant and outside-only terms onto any dense pair op in the group
        {
            QForm cpart;
            std::vector<int> csel;
            bool ok = true;
            cpart.cst = F.cst;
            for (auto &kv : F.lin)
                if (!((S >> kv.first) & 1)) {
                    cpart.lin[kv.first] = kv.second;
                    if (!((sel_ok >> kv.first) & 1)) ok = false;
                    if (std::find(csel.begin(), csel.end(), kv.first) == csel.end()) csel.push_back(kv.first);
                }
            for (auto &kv : F.quad) {
                const int x = kv.first.first, y = kv.first.second;
                if (((S >> x) & 1) || ((S >> y) & 1)) continue;
                cpart.quad[kv.first] = kv.second;
                for (int q : {x, y}) {
                    if (!((sel_ok >> q) & 1)) ok = false;
                    if (std::find(csel.begin(), csel.end(), q) == csel.end()) csel.push_back(q);
                }
            }
            if (ok && !cpart.trivial()) {
                int best = -1, bn = 99;
                for (size_t i = 0; i < ops.size(); ++i) {
                    if (!is_pair_dense(ops[i])) continue;
                    std::vector<int> s2 = ops[i].sel;
                    for (int x : csel)
                        if (std::find(s2.begin(), s2.end(), x) == s2.end()) s2.push_back(x);
                    if ((int)s2.size() < bn) { bn = (int)s2.size(); best = (int)i; }
                }
                if (best >= 0 && bn <= kMaxSel) {
                    fold_diag_into(ops[best], cpart, csel, true);   // scalars commute: any side
                    F.cst = 0;
                    for (auto &kv : cpart.lin) F.lin.erase(kv.first);
                    for (auto &kv : cpart.quad) F.quad.erase(kv.first);
                }
            }
        }
        ops[k].qmask = F.qubits();
    }
    for (size_t k = 0; k < ops.size();) {
        if (ops[k].type == OP_DIAG && ops[k].form.trivial()) ops.erase(ops.begin() + (long)k);
        else ++k;
    }
}

static void merge_variant_chains(FOp &grp, uint64_t S, int nl) {
    // selectors on global (rank) bits are encoded relative to bit 32 (pass_format.h)
    const uint64_t sel_ok = ~0ull;   // global-bit selectors are resolved per rank at encode time
    (void)nl;
    std::vector<FOp> &ops = grp.subs;
    for (size_t i = 0; i < ops.size(); ++i) {
        if (ops[i].type != OP_DENSE || ops[i].tg.size() != 2) continue;
        const int a = ops[i].tg[0], b = ops[i].tg[1];
        const uint64_t P = (1ull << a) | (1ull << b);
        // previous op touching P
        int j = (int)i - 1;
        for (; j >= 0; --j) {
            const FOp &o = ops[j];
            if (o.type == OP_DIAG) continue;
            if (o.qmask & P) break;
        }
        if (j < 0 || ops[j].type != OP_DENSE || ops[j].tg.size() != 2 || ops[j].dmask != P) continue;
        // the P-parts of the diagonals in between must couple P only to bits outside the tile
        bool ok = true;
        std::vector<int> sel = ops[j].sel;
        std::vector<QForm> parts;
        for (size_t k = j + 1; k < i && ok; ++k) {
            const FOp &o = ops[k];
            if (o.type != OP_DIAG) continue;
            QForm part;
            for (auto &kv : o.form.lin)
                if ((P >> kv.first) & 1) part.lin[kv.first] += kv.second;
            for (auto &kv : o.form.quad) {
                const int x = kv.first.first, y = kv.first.second;
                const bool px = (P >> x) & 1, py = (P >> y) & 1;
                if (!px && !py) continue;
                if (px && py) { part.quad[kv.first] += kv.second; continue; }
                const int other = px ? y : x;
                if ((S >> other) & 1) { ok = false; break; }        // varies inside the tile
                if (!((sel_ok >> other) & 1)) { ok = false; break; }
                part.quad[kv.first] += kv.second;
                if (std::find(sel.begin(), sel.end(), other) == sel.end()) sel.push_back(other);
            }
            parts.push_back(part);
        }
        for (int x : ops[i].sel)
            if (std::find(sel.begin(), sel.end(), x) == sel.end()) sel.push_back(x);
        if (!ok || (int)sel.size() > kMaxSel) continue;
        // the per-tile constant parts of those diagonals (constant, terms on bits outside the
        // tile only) ride along when the selector budget allows: they are scalars per tile
        std::vector<bool> take_const(i, false);
        {
            size_t pi = 0;
            for (size_t k = j + 1; k < i; ++k) {
                const FOp &o = ops[k];
                if (o.type != OP_DIAG) continue;
                std::vector<int> s2 = sel;
                auto need = [&](int q) {
                    if (std::find(s2.begin(), s2.end(), q) == s2.end()) s2.push_back(q);
                };
                bool any = o.form.cst != 0;
                for (auto &kv : o.form.lin)
                    if (!((S >> kv.first) & 1)) { need(kv.first); any = true; if (!((sel_ok >> kv.first) & 1)) any = false, s2.assign(kMaxSel + 1, 0); }
                for (auto &kv : o.form.quad)
                    if (!((S >> kv.first.first) & 1) && !((S >> kv.first.second) & 1)) {
                        need(kv.first.first);
                        need(kv.first.second);
                        any = true;
                        if (!((sel_ok >> kv.first.first) & 1) || !((sel_ok >> kv.first.second) & 1))
                            s2.assign(kMaxSel + 1, 0);                 // cannot encode: leave in place
                    }
                if (any && (int)s2.size() <= kMaxSel) {
                    sel = s2;
                    take_const[k] = true;
                    QForm &part = parts[pi];
                    part.cst += o.form.cst;
                    for (auto &kv : o.form.lin)
                        if (!((S >> kv.first) & 1)) part.lin[kv.first] += kv.second;
                    for (auto &kv : o.form.quad)
                        if (!((S >> kv.first.first) & 1) && !((S >> kv.first.second) & 1)) part.quad[kv.first] += kv.second;
                }
                ++pi;
            }
        }
        std::sort(sel.begin(), sel.end());
        const int nv = 1 << (int)sel.size();
        auto variant_of = [&](const FOp &o, int v) -> const std::vector<cd> & {
            if (o.Mv.empty()) return o.M;
            int w = 0;
            for (size_t q = 0; q < o.sel.size(); ++q) {
                const size_t pos = std::find(sel.begin(), sel.end(), o.sel[q]) - sel.begin();
                if ((v >> pos) & 1) w |= 1 << q;
            }
            return o.Mv[(size_t)w];
        };
        std::vector<std::vector<cd>> Mv((size_t)nv);
        for (int v = 0; v < nv; ++v) {
            std::vector<cd> M = variant_of(ops[j], v);
            for (const QForm &part : parts) M = matmul(diag_on_pair(part, a, b, sel, v), M, 4);
            Mv[(size_t)v] = matmul(variant_of(ops[i], v), M, 4);
        }
        // strip the moved parts from the diagonals; drop diagonals that became empty
        const uint64_t out = ~S;
        for (size_t k = j + 1; k < i; ++k) {
            FOp &o = ops[k];
            if (o.type != OP_DIAG) continue;
            const bool tc = take_const[k];
            if (tc) o.form.cst = 0;
            for (auto it = o.form.lin.begin(); it != o.form.lin.end();) {
                const bool mv = ((P >> it->first) & 1) || (tc && ((out >> it->first) & 1));
                it = mv ? o.form.lin.erase(it) : std::next(it);
            }
            for (auto it = o.form.quad.begin(); it != o.form.quad.end();) {
                const int x = it->first.first, y = it->first.second;
                const bool mv = ((P >> x) & 1) || ((P >> y) & 1) || (tc && ((out >> x) & 1) && ((out >> y) & 1));
                it = mv ? o.form.quad.erase(it) : std::next(it);
            }
            o.qmask = o.form.qubits();
        }
        FOp merged = ops[i];
        merged.Mv = Mv;
        merged.sel = sel;
        merged.M = Mv[0];
        ops[i] = merged;
        ops.erase(ops.begin() + j);
        --i;
        for (size_t k = 0; k < ops.size();) {
            if (ops[k].type == OP_DIAG && ops[k].form.trivial()) {
                ops.erase(ops.begin() + (long)k);
                if (k <= i) --i;
            } else if (k > 0 && ops[k].type == OP_DIAG && ops[k - 1].type == OP_DIAG) {
                ops[k - 1].form.add(ops[k].form);             // adjacent diagonals: one sub-op
                ops[k - 1].qmask = ops[k - 1].form.qubits();
                ops.erase(ops.begin() + (long)k);
                if (k <= i) --i;
            } else ++k;
        }
    }
}

// Algorithmic floating-point work per amplitude: a k-qubit
// dense op costs 8 * 2^k flops (2^k complex multiply-adds), a diagonal phase
// one complex multiply (6), a CNOT none.
double pass_flops_per_amp(const std::vector<FOp> &ops) {
    double f = 0;
    for (const FOp &o : ops) {
        if (o.type == OP_GROUP) f += pass_flops_per_amp(o.subs);
        else if (o.type == OP_DENSE) f += 8.0 * (1 << o.tg.size());
        else if (o.type == OP_DIAG) f += 6.0;
    }
    return f;
}

// Tensor-core programs (complex64, tiles of <= 12 bits): the part of a group's
// diagonal sub-op that differs between the vectors of a tile (terms on a V-bit:
// an in-tile bit outside the group's registers) is sunk to the END of the group's
// program when no later sub-op acts non-diagonally on its register bits (diagonal
// terms commute with every op that acts on their bits only diagonally; V-bits and
// outside bits are never targets inside a group).  What stays is the same for every
// vector, so runs of matrices separated only by such diagonals merge into one
// operator step, and the sunk terms become one trailing register (E) step.
// Returns false (and leaves the group unchanged) when nothing moves.
static bool sink_v_terms(FOp &grp, uint64_t S) {
    // terms on a bit outside the tile (the tile base) are per-tile factors of the same kind:
    // sunk too, the operators of the group stop depending on the tile base (no per-tile
    // rebuild; QFT groups of c3: H's + their register-register phases = one constant operator)
    static const bool sink_out = !(getenv("STV_SINK_OUT") && !atoi(getenv("STV_SINK_OUT")));
    const uint64_t T = grp.T, V = sink_out ? ~T : (S & ~T);
    std::vector<FOp> subs = grp.subs;
    QForm sunk;
    bool moved = false;
    uint64_t blocked = 0;   // register bits acted on non-diagonally after position k
    for (size_t k = subs.size(); k-- > 0;) {
        FOp &o = subs[k];
        if (o.type == OP_DIAG) {
            QForm vpart, rest;
            rest.cst = o.form.cst;
            for (auto &kv : o.form.lin) ((V >> kv.first) & 1 ? vpart.lin : rest.lin)[kv.first] = kv.second;
            for (auto &kv : o.form.quad) {
                const bool hv = ((V >> kv.first.first) & 1) || ((V >> kv.first.second) & 1);
                (hv ? vpart.quad : rest.quad)[kv.first] = kv.second;
            }
            if (!vpart.trivial() && !(vpart.qubits() & T & blocked) && !(k + 1 == subs.size() && !moved)) {
                sunk.add(vpart);
                o.form = rest;
                o.qmask = rest.qubits();
                moved = true;
            }
        } else if (o.type == OP_DENSE) {
            for (int b : o.tg) blocked |= 1ull << b;
        } else if (o.type == OP_CNOT) {
            blocked |= 1ull << o.t;
        }
    }
    if (!moved) return false;
    std::vector<FOp> out;
    for (FOp &o : subs)
        if (!(o.type == OP_DIAG && o.form.trivial())) out.push_back(std::move(o));
    if (!out.empty() && out.back().type == OP_DIAG) {   // merge with a trailing diagonal
        out.back().form.add(sunk);
        out.back().qmask = out.back().form.qubits();
    } else {
        FOp d;
        d.type = OP_DIAG;
        d.form = sunk;
        d.qmask = sunk.qubits();
        out.push_back(std::move(d));
    }
    grp.subs = std::move(out);
    return true;
}

Plan build_plan(int n, int n_global, int amp_bytes, const std::vector<PGate> &pg_virtual,
                const PlanOptions &opt, int *sigma) {
    Plan plan;
    plan.n = n;
    plan.n_global = n_global;
    plan.flags = opt.flags;
    const int nl = n - n_global;
    const uint64_t local_mask = nl >= 64 ? ~0ull : ((1ull << nl) - 1);
    const uint64_t all_mask = n >= 64 ? ~0ull : ((1ull << n) - 1);
    const uint64_t low_mask = (1ull << opt.low_bits) - 1;
    const bool one_gate = opt.flags & SV_OPT_ONE_GATE;
    const bool no_reorder = opt.flags & SV_OPT_NO_REORDER;
    const bool fold = !(opt.flags & SV_OPT_NO_DIAG_FOLD);
    const size_t G = pg_virtual.size();
    std::vector<char> done(G, 0);
    size_t first = 0;
    const double amp_pass_bytes = 2.0 * amp_bytes * std::ldexp(1.0, nl);   // R+W per rank
    // the group pass record is a kernel parameter (<= STV_REC_PARAM_BYTES); its
    // diag tables share the CTA's shared memory with 2 tile stages: keep three
    // CTAs per SM when the tiles allow it
    const size_t tile_b = (size_t)amp_bytes << opt.tile_bits;
    const size_t rec_limit = std::min(kMaxRecBytes, (size_t)STV_REC_PARAM_BYTES);
    // (diagonal-heavy passes, e.g. the QFT of c3, trade the third CTA for full-size tiles:
    // a 16 KB table area measured best on c3, 306 vs 506 ms/circuit at 8 KB; 24 KB once the
    // per-tile table build spread its terms over the lanes: 7 passes instead of 9, 242 -> 229 ms)
    size_t tab_limit = 24 * 1024;
    if (const char *e = getenv("STV_TAB_LIMIT")) tab_limit = (size_t)atoi(e);

    while (true) {
        while (first < G && done[first]) ++first;
        if (first >= G) break;
        PPass pass;
        pass.kind = PASS_TILE;
        uint64_t S = low_mask & local_mask;
        uint64_t blockedAll = 0, blockedDense = 0;
        std::vector<PGate> pgates;               // absorbed gates (actual bits), in order
        OpsEval cur;
        for (size_t i = first; i < G; ++i) {
            if (done[i]) continue;
            if ((blockedAll & all_mask) == all_mask) break;
            PGate g = map_gate(pg_virtual[i], sigma);
            const uint64_t qm = g.qmask(), dm = g.dmask();
            bool ok = !(qm & blockedAll) && !(dm & blockedDense) && !(dm & ~local_mask);
            uint64_t need = dm & ~S;
            if (ok && __builtin_popcountll(S | need) > opt.tile_bits) ok = false;
            if (ok && one_gate && !pgates.empty()) ok = false;
            if (ok) {
                pgates.push_back(g);
                const bool incremental = cur.grouped && need == 0;   // tile set unchanged
                if (incremental) add_gate(cur, g, S, opt, amp_bytes);
                else {
                    OpsEval t = make_ops(pgates, S | need, opt, amp_bytes);
                    std::swap(cur, t);
                }
                if (pgates.size() > 1 &&
                    (cur.cost > opt.budget || cur.rec > rec_limit || cur.tab > tab_limit ||
                     cur.ntab > STV_MAX_TABLES)) {
                    ok = false;
                    pgates.pop_back();
                    cur = make_ops(pgates, S, opt, amp_bytes);        // rare: rebuild without g
                }
            }
            if (!ok) {
                blockedAll |= dm;
                blockedDense |= qm & ~dm;
                if (no_reorder) break;
                continue;
            }
            S |= need;
            done[i] = 1;
            pass.gates.push_back(g.src);
        }
        pass.ops = cur.ops;
        if (pass.ops.empty()) {
            // frontier needs a global qubit as a non-diagonal target: remap
            // (SURVEY.md 8(e)).  Needed global bits from the earliest gates.
            uint64_t gneed = 0;
            for (size_t i = first; i < G && __builtin_popcountll(gneed) < n_global; ++i) {
                if (done[i]) continue;
                PGate g = map_gate(pg_virtual[i], sigma);
                gneed |= g.dmask() & ~local_mask;
                if (i > first + 64 && gneed) break;
            }
            if (!gneed) {   // cannot happen with tile_bits >= 2; guard against a stall
                throw std::runtime_error("planner stall");
            }
            // Belady: local victims whose next non-diagonal use is furthest away
            std::vector<std::pair<size_t, int>> cand;
            for (int b = opt.low_bits; b < nl; ++b) {
                size_t next = G + 1;
                for (size_t i = first; i < G; ++i) {
                    if (done[i]) continue;
                    PGate g = map_gate(pg_virtual[i], sigma);
                    if (g.dmask() >> b & 1) { next = i; break; }
                }
                cand.push_back({next, b});
            }
            std::sort(cand.begin(), cand.end(), [](auto &a, auto &b) {
                return a.first != b.first ? a.first > b.first : a.second > b.second;
            });
            PPass rp;
            rp.kind = PASS_REMAP;
            size_t ci = 0;
            for (int gb : bits_of(gneed)) {
                int lb = cand[ci++].second;
                rp.swaps.push_back({gb, lb});
                // the virtual bits at actual positions gb and lb exchange places
                for (int v = 0; v < n; ++v) {
                    if (sigma[v] == gb) sigma[v] = lb;
                    else if (sigma[v] == lb) sigma[v] = gb;
                }
            }
            plan.alg_bytes += (double)rp.swaps.size() > 0 ? amp_pass_bytes * (1.0 - std::ldexp(1.0, -(int)rp.swaps.size())) : 0;
            plan.passes.push_back(rp);
            continue;
        }
        // pass kind: standalone streaming kernels when no tile is needed
        bool all_diag = true;
        for (auto &g : pgates) all_diag &= (g.type == GType::DIAG);
        if (all_diag) {
            pass.kind = PASS_DIAG;
            FOp merged;
            merged.type = OP_DIAG;
            for (auto &g : pgates) { merged.form.add(g.form); merged.qmask |= g.qmask(); }
            pass.ops.assign(1, merged);
            pass.S = 0;
            // skip-write: unchanged amplitudes are not written
            plan.alg_bytes += amp_pass_bytes / 2 * 1.5;
        } else if (pgates.size() == 1 && pgates[0].type == GType::CNOT) {
            pass.kind = PASS_CNOT;
            FOp c;
            c.type = OP_CNOT;
            c.c = pgates[0].q[0];
            c.t = pgates[0].q[1];
            pass.ops.assign(1, c);
            pass.S = 0;
            plan.alg_bytes += amp_pass_bytes / 2;
        } else {
            // pad the tile to full size with the lowest free local bits: bits no
            // gate of the pass touches cost nothing and lengthen the contiguous
            // runs (then any bit, re-grouping with the final tile)
            uint64_t touched = 0;
            for (auto &g : pgates) touched |= g.qmask();
            for (int b = 0; b < nl && __builtin_popcountll(S) < opt.tile_bits; ++b)
                if (!((touched >> b) & 1)) S |= 1ull << b;
            const uint64_t S0 = S;
            for (int b = 0; b < nl && __builtin_popcountll(S) < opt.tile_bits; ++b) S |= 1ull << b;
            if (S != S0) {
                OpsEval fin = make_ops(pgates, S, opt, amp_bytes);
                if (fin.rec <= rec_limit && fin.tab <= tab_limit && fin.ntab <= STV_MAX_TABLES) pass.ops = fin.ops;
                else S = S0;
            }
            pass.S = S;
            if (!(opt.flags & SV_OPT_NO_VARIANTS)) {
                bool grouped = !pass.ops.empty();
                for (FOp &o : pass.ops) grouped &= o.type == OP_GROUP;
                if (grouped) relocate_v_terms(pass.ops, S);
            }
            if (!(opt.flags & SV_OPT_NO_VARIANTS))
                for (FOp &o : pass.ops)
                    if (o.type == OP_GROUP) {
                        absorb_diagonals(o, S, nl);
                        merge_variant_chains(o, S, nl);
                    }
            // tensor-core programs: V-bit diagonal terms sunk to the end of each group (kept
            // only if the pass's tables still fit)
            if (amp_bytes == 8 && !(opt.flags & (SV_OPT_NO_TC | SV_OPT_NO_SINK)) && __builtin_popcountll(S) <= 12) {
                std::vector<FOp> trial = pass.ops;
                bool any = false;
                for (FOp &o : trial)
                    if (o.type == OP_GROUP) any |= sink_v_terms(o, S);
                if (any) {
                    OpsEval ev;
                    ev.ops = trial;
                    ev.grouped = true;
                    tally(ev, amp_bytes, S);
                    if (ev.rec <= rec_limit && ev.tab <= tab_limit && ev.ntab <= STV_MAX_TABLES) pass.ops = trial;
                }
            }
            plan.alg_bytes += amp_pass_bytes;
            plan.alg_flops += pass_flops_per_amp(pass.ops) * std::ldexp(1.0, nl);
        }
        plan.passes.push_back(pass);
    }
    for (int v = 0; v < 64; ++v) plan.sigma_out[v] = v < n ? sigma[v] : v;
    return plan;
}

// ---------------------------------------------------------------------------
// encoding for the device (pass_format.h)
// ---------------------------------------------------------------------------
static void put(std::vector<uint8_t> &b, const void *p, size_t n) {
    const uint8_t *c = (const uint8_t *)p;
    b.insert(b.end(), c, c + n);
}
static void align(std::vector<uint8_t> &b, size_t a) {
    while (b.size() % a) b.push_back(0);
}

// Diag record relative to tile: positions pos[0..S) = physical bits (ascending
// map loc[]), the rest are "outside" (per-tile constants).
static void encode_diag(std::vector<uint8_t> &b, size_t rec_at, const QForm &f, const int *loc, int S) {
    StvDiag d;
    std::memset(&d, 0, sizeof(d));
    d.cst = f.cst;
    std::vector<StvTerm> cross, olin, oquad;
    bool quarter = (f.cst & ((1ull << 62) - 1)) == 0;
    for (auto &kv : f.lin) {
        quarter &= (kv.second & ((1ull << 62) - 1)) == 0;
        int l = loc[kv.first];
        if (l >= 0) d.lin[l] += kv.second;
        else olin.push_back({kv.first, -1, kv.second});
    }
    for (auto &kv : f.quad) {
        quarter &= (kv.second & ((1ull << 62) - 1)) == 0;
        int a = kv.first.first, c = kv.first.second;
        int la = loc[a], lc = loc[c];
        if (la >= 0 && lc >= 0) { d.A[la][lc] += kv.second; d.A[lc][la] += kv.second; }
        else if (la >= 0) cross.push_back({la, c, kv.second});
        else if (lc >= 0) cross.push_back({lc, a, kv.second});
        else oquad.push_back({a, c, kv.second});
    }
    d.all_quarter = quarter ? 1 : 0;
    std::stable_sort(cross.begin(), cross.end(), [](const StvTerm &x, const StvTerm &y) { return x.a < y.a; });
    for (int q = 0, k = 0; q <= S + 1 && q < STV_MAX_TILE_BITS + 2; ++q) {
        while (k < (int)cross.size() && cross[k].a < q) ++k;
        d.cross_start[q] = k;
    }
    d.n_cross = (int)cross.size();
    d.n_olin = (int)olin.size();
    d.n_oquad = (int)oquad.size();
    size_t off = sizeof(StvDiag);
    d.cross_off = (uint32_t)off; off += cross.size() * sizeof(StvTerm);
    d.olin_off = (uint32_t)off; off += olin.size() * sizeof(StvTerm);
    d.oquad_off = (uint32_t)off;
    std::memcpy(&b[rec_at], &d, sizeof(d));
    put(b, cross.data(), cross.size() * sizeof(StvTerm));
    put(b, olin.data(), olin.size() * sizeof(StvTerm));
    put(b, oquad.data(), oquad.size() * sizeof(StvTerm));
}

// Shared-memory slot of tile amplitude i under the chunk swizzle of
// pass_format.h (linear over GF(2)).
// Tile swizzle of the pass being encoded: the group pass's XOR pattern H (kSwzH), or for
// tensor-core passes staged by TMA the SWIZZLE_128B pattern H(x) = x & 7 (16-B chunk j of
// each 128-B line stored at j ^ (line mod 8); pass_format.h StvPass.swz_tma).
static thread_local bool g_swz_tma = false;
static uint32_t swz_hash(uint32_t x) {
    if (g_swz_tma) return x & 7u;
    return (uint32_t)(__builtin_popcount(x & kSwzM0) & 1) | ((uint32_t)(__builtin_popcount(x & kSwzM1) & 1) << 1) |
           ((uint32_t)(__builtin_popcount(x & kSwzM2) & 1) << 2);
}
static uint32_t swz_amp(uint32_t i, bool c128) {
    if (c128) return i ^ swz_hash(i >> 3);
    const uint32_t c = i >> 1;
    return (((c ^ swz_hash(c >> 3))) << 1) | (i & 1);
}

// bank vector (3 bits) of tile position p: which 16-B bank group a chunk bit selects
static uint32_t bank_vec(int p, bool c128) {
    const int j = c128 ? p : p - 1;          // chunk bit
    if (j < 0) return 0;
    if (j < 3) return 1u << j;
    if (g_swz_tma) return j < 6 ? (1u << (j - 3)) : 0u;
    return kSwzH[j - 3];
}

// Order of a group's vector bits: lane bits 0..2 (LDS.128 phases of 8 lanes)
// get positions with linearly independent bank vectors; a complex64 group
// without position 0 uses 8-B accesses (16-lane phases), so position 0 leads.
static std::vector<int> vector_bit_order(const std::vector<int> &pos, int S, bool c128, int avoid = -1) {
    std::vector<int> R, head, order;
    for (int q = 0; q < S; ++q)
        if (std::find(pos.begin(), pos.end(), q) == pos.end()) R.push_back(q);
    if (!c128 && pos[0] != 0 && avoid != 0) head.push_back(0);
    std::vector<uint32_t> basis;
    auto reduce = [&](uint32_t v) {
        for (uint32_t b : basis) v = std::min(v, v ^ b);
        return v;
    };
    // lane bits: 3 positions with independent bank vectors (`avoid`, a position wanted as
    // vector bit 7, is used only if no other position completes the basis)
    for (int pass = 0; pass < 2; ++pass)
        for (int q : R) {
            if (basis.size() >= 3) break;
            if (!c128 && q == 0) continue;
            if ((q == avoid) != (pass == 1)) continue;
            const uint32_t v = reduce(bank_vec(q, c128));
            if (v) { basis.push_back(v); head.push_back(q); }
        }
    if (!c128 && pos[0] != 0 && avoid == 0) head.insert(head.begin(), 0);   // amplitude bit 0 is unavoidable
    order = head;
    for (int q : R)
        if (std::find(head.begin(), head.end(), q) == head.end()) order.push_back(q);
    return order;
}

// One per-tile phase table of a group diagonal sub-op (pass_format.h StvDTab).
struct GroupTable {
    std::vector<int> vpos;           // tile positions of its V-bits (<= STV_MAX_VBITS, or _H for half)
    std::vector<uint64_t> stat;      // static phases, index l | r << 4 (half: l' | r << 3)
    std::vector<StvTerm> terms;      // per-tile terms
    int half = -1;                   // >= 0: half table on local bit `half`
};

// A diagonal whose every term contains local bit j (no constant) and that has at
// most STV_MAX_VBITS_H V-bits: one half table (pass_format.h).
static bool half_table(const QForm &f, const std::vector<int> &pos, const int *loc, GroupTable &gt) {
    if (f.cst != 0) return false;
    auto local = [&](int phys) -> int {
        if (loc[phys] < 0) return -1;
        auto it = std::find(pos.begin(), pos.end(), loc[phys]);
        return it == pos.end() ? -1 : (int)(it - pos.begin());
    };
    auto is_v = [&](int phys) { return loc[phys] >= 0 && local(phys) < 0; };
    for (int j = 0; j < 4; ++j) {
        const int pj = [&] { for (auto &kv : f.lin) if (local(kv.first) == j) return kv.first;
                             for (auto &kv : f.quad) { if (local(kv.first.first) == j) return kv.first.first;
                                                       if (local(kv.first.second) == j) return kv.first.second; }
                             return -1; }();
        if (pj < 0) continue;
        bool ok = true;
        std::vector<int> vp;
        for (auto &kv : f.lin) ok &= kv.first == pj;
        for (auto &kv : f.quad) {
            const int x = kv.first.first, y = kv.first.second;
            if (x != pj && y != pj) { ok = false; break; }
            const int o = x == pj ? y : x;
            if (is_v(o) && std::find(vp.begin(), vp.end(), loc[o]) == vp.end()) vp.push_back(loc[o]);
        }
        if (!ok || (int)vp.size() > STV_MAX_VBITS_H) continue;
        std::sort(vp.begin(), vp.end());
        gt.vpos = vp;
        gt.half = j;
        const int m = (int)vp.size();
        gt.stat.assign((size_t)8 << m, 0);
        // index bits: 0..2 = the other local bits ascending, 3.. = V-bits
        auto ibit = [&](int phys) -> int {
            const int l = local(phys);
            if (l >= 0) return l < j ? l : l - 1;
            return 3 + (int)(std::find(vp.begin(), vp.end(), loc[phys]) - vp.begin());
        };
        for (auto &kv : f.lin)
            for (auto &e : gt.stat) e += kv.second;                 // l_j = 1 for every entry
        for (auto &kv : f.quad) {
            const int x = kv.first.first, y = kv.first.second;
            const int o = x == pj ? y : x;
            if (loc[o] < 0) { gt.terms.push_back({-1, o, kv.second}); continue; }   // per-tile constant
            const int b = ibit(o);
            for (size_t e = 0; e < gt.stat.size(); ++e)
                if ((e >> b) & 1) gt.stat[e] += kv.second;
        }
        return true;
    }
    return false;
}

// Split a group's diagonal form into tables of <= STV_MAX_VBITS V-bits each
// (diagonal terms commute and add, so the split is exact).
// Several half tables for a diagonal whose every term contains one group bit j but
// that has more than STV_MAX_VBITS_H V-bits: terms partitioned by their V-bit.
static bool half_tables_split(const QForm &f, const std::vector<int> &pos, const int *loc,
                              std::vector<GroupTable> &out) {
    if (f.cst != 0) return false;
    auto local = [&](int phys) -> int {
        if (loc[phys] < 0) return -1;
        auto it = std::find(pos.begin(), pos.end(), loc[phys]);
        return it == pos.end() ? -1 : (int)(it - pos.begin());
    };
    for (int j = 0; j < 4; ++j) {
        int pj = -1;
        for (auto &kv : f.quad)
            for (int q : {kv.first.first, kv.first.second})
                if (local(q) == j) pj = q;
        for (auto &kv : f.lin)
            if (local(kv.first) == j) pj = kv.first;
        if (pj < 0) continue;
        bool ok = true;
        for (auto &kv : f.lin) ok &= kv.first == pj;
        for (auto &kv : f.quad) ok &= kv.first.first == pj || kv.first.second == pj;
        if (!ok) continue;
        // chunks of terms with <= STV_MAX_VBITS_H distinct V-partners each
        std::vector<QForm> parts(1);
        std::vector<std::vector<int>> vs(1);
        parts[0].lin = f.lin;
        for (auto &kv : f.quad) {
            const int o = kv.first.first == pj ? kv.first.second : kv.first.first;
            const bool v = loc[o] >= 0 && local(o) < 0;
            size_t t = 0;
            if (v) {
                for (; t < parts.size(); ++t) {
                    const bool has = std::find(vs[t].begin(), vs[t].end(), o) != vs[t].end();
                    if (has || (int)vs[t].size() < STV_MAX_VBITS_H) {
                        if (!has) vs[t].push_back(o);
                        break;
                    }
                }
                if (t == parts.size()) { parts.emplace_back(); vs.push_back({o}); }
            }
            parts[t].quad[kv.first] = kv.second;
        }
        for (const QForm &q : parts) {
            GroupTable gt;
            if (!half_table(q, pos, loc, gt)) return false;
            out.push_back(gt);
        }
        return true;
    }
    return false;
}

static std::vector<GroupTable> split_group_diag(const QForm &f, const std::vector<int> &pos, const int *loc) {
    {
        GroupTable gt;
        if (half_table(f, pos, loc, gt)) return {gt};
        std::vector<GroupTable> hs;
        if (half_tables_split(f, pos, loc, hs)) return hs;
    }
    struct Item { int x, y; uint64_t ang; };   // y = -1: linear term on x
    std::vector<Item> items;
    for (auto &kv : f.lin) items.push_back({kv.first, -1, kv.second});
    for (auto &kv : f.quad) items.push_back({kv.first.first, kv.first.second, kv.second});
    auto is_v = [&](int phys) {
        return loc[phys] >= 0 && std::find(pos.begin(), pos.end(), loc[phys]) == pos.end();
    };
    std::vector<std::vector<int>> vsets;       // per table: V tile positions
    std::vector<std::vector<Item>> members;
    for (const Item &it : items) {
        std::vector<int> need;
        for (int q : {it.x, it.y})
            if (q >= 0 && is_v(q)) need.push_back(loc[q]);
        size_t t = 0;
        for (; t < vsets.size(); ++t) {
            std::vector<int> u = vsets[t];
            for (int v : need)
                if (std::find(u.begin(), u.end(), v) == u.end()) u.push_back(v);
            if ((int)u.size() <= STV_MAX_VBITS) { vsets[t] = u; break; }
        }
        if (t == vsets.size()) { vsets.push_back(need); members.emplace_back(); }
        members[t].push_back(it);
    }
    if (vsets.empty()) { vsets.emplace_back(); members.emplace_back(); }   // constant-only form
    std::vector<GroupTable> out;
    for (size_t t = 0; t < vsets.size(); ++t) {
        GroupTable gt;
        gt.vpos = vsets[t];
        std::sort(gt.vpos.begin(), gt.vpos.end());
        const int m = (int)gt.vpos.size();
        // index bit of a physical qubit in this table (-1: outside the tile)
        auto ibit = [&](int phys) -> int {
            if (loc[phys] < 0) return -1;
            auto it = std::find(pos.begin(), pos.end(), loc[phys]);
            if (it != pos.end()) return (int)(it - pos.begin());
            return 4 + (int)(std::find(gt.vpos.begin(), gt.vpos.end(), loc[phys]) - gt.vpos.begin());
        };
        gt.stat.assign((size_t)16 << m, t == 0 ? f.cst : 0);
        for (const Item &it : members[t]) {
            const int bx = ibit(it.x), by = it.y >= 0 ? ibit(it.y) : -1;
            if (it.y < 0) {
                if (bx >= 0) {
                    for (size_t e = 0; e < gt.stat.size(); ++e)
                        if ((e >> bx) & 1) gt.stat[e] += it.ang;
                } else gt.terms.push_back({-1, it.x, it.ang});
            } else if (bx >= 0 && by >= 0) {
                for (size_t e = 0; e < gt.stat.size(); ++e)
                    if (((e >> bx) & 1) && ((e >> by) & 1)) gt.stat[e] += it.ang;
            } else if (bx >= 0) gt.terms.push_back({bx, it.y, it.ang});
            else if (by >= 0) gt.terms.push_back({by, it.x, it.ang});
            else gt.terms.push_back({-2 - it.x, it.y, it.ang});
        }
        out.push_back(gt);
    }
    return out;
}

// ---------------------------------------------------------------------------
// Tensor-core step plan of a grouped complex64 pass (pass_format.h StvTcStep,
// tc_pass.cuh).  Each group's final sub-op program is cut into maximal runs of
// sub-ops that act identically on every vector of a tile ("foldable": matrices,
// per-tile variants, CNOTs without a V-bit control, diagonal tables without
// V-bits) and the rest.  A foldable run whose FMA cost reaches STV_TC_MIN
// (FFMA2-equivalents per vector, default 150: STV_TC_MIN sweeps with tools/ab_env.sh; cheaper runs stay on
// the registers) becomes an M step: one 16 x 16 operator applied with tcgen05.mma.
// ---------------------------------------------------------------------------
static int nth_set_bit(uint64_t m, int i) {
    for (int k = 0; k < 64; ++k)
        if ((m >> k) & 1) {
            if (i-- == 0) return k;
        }
    return -1;
}

static void encode_tc_steps(std::vector<uint8_t> &b, size_t at, StvPass &hd, const std::vector<StvGroup> &grecs,
                            const std::vector<StvDTab> &tabs) {
    static const double tc_min = getenv("STV_TC_MIN") ? atof(getenv("STV_TC_MIN")) : 150.0;
    uint32_t bvraw = 0;   // raw tile offset of the current group's vector bit 7 (its TMEM block), or 0
    // 0: varies between the vectors of a block (E step); 1: uniform over the tile; 2: uniform
    // within each block (a per-block operator variant: depends only on vector bit 7)
    auto fold_kind = [&](const StvSub &x) -> int {
        const int c = x.code & 0xff;
        if (c >= SUBC_CNOT && c < SUBC_DIAG) {
            const uint32_t raw = x.ctl & 0xffffu;
            return raw == 0 ? 1 : (bvraw && raw == bvraw) ? 2 : 0;
        }
        if (c == SUBC_DIAG || (c >= SUBC_DIAGH && c < SUBC_DIAGH + 4)) {
            const StvDTab &d = tabs[x.arg];
            return d.m == 0 ? 1 : (bvraw && d.m == 1 && d.vraw[0] == bvraw) ? 2 : 0;
        }
        return 1;
    };
    auto foldable = [&](const StvSub &x) { return fold_kind(x) != 0; };
    // per sub-op dispatch on the registers (uniform branch, operand loads): long runs of cheap
    // sub-ops (the QFT's Hadamards between half tables, c3) cost more than their arithmetic
    static const double dispatch_cost = getenv("STV_TC_SUBOP") ? atof(getenv("STV_TC_SUBOP")) : 16.0;
    auto arith = [&](const StvSub &x) -> double {   // FFMA2-equivalents per 16-amplitude vector
        const int c = x.code & 0xff;
        if (c < SUBC_U2) return 32;
        if (c < SUBC_CNOT) return 128;
        if (c < SUBC_DIAG) return 16;
        if (c == SUBC_DIAG) return 40;
        if (c < SUBC_DIAGH) return 128;          // U2V
        if (c < SUBC_U2X2) return 20;            // half table
        if (c < SUBC_U1R) return 256;            // two U2
        if (c < SUBC_U2R) return 16;
        return 64;
    };
    auto cost = [&](const StvSub &x) -> double { return dispatch_cost + arith(x); };
    auto sel_bits = [&](uint32_t w, uint64_t &dep) {   // 3 x 5-bit tile-ordinal selectors
        for (int i = 0; i < 3; ++i) {
            const uint32_t sl = (w >> (5 * i)) & 31u;
            if (sl != 31u) {
                const int pb = nth_set_bit(hd.out_mask, (int)sl);
                if (pb >= 0) dep |= 1ull << pb;
            }
        }
    };
    auto depends = [&](const StvSub &x) -> uint64_t {   // tile-base bits the op's action depends on
        const int c = x.code & 0xff;
        uint64_t dep = 0;
        if (c >= SUBC_U2V && c < SUBC_U2V + 6) sel_bits((uint32_t)x.code >> 8, dep);
        if (c >= SUBC_U2X2 && c < SUBC_U2X2 + 3) {
            sel_bits((uint32_t)x.code >> 8, dep);
            sel_bits(x.pad, dep);
        }
        if (c >= SUBC_CNOT && c < SUBC_DIAG && (x.ctl >> 16)) dep |= 1ull << ((x.ctl >> 16) - 1);
        if (c == SUBC_DIAG || (c >= SUBC_DIAGH && c < SUBC_DIAGH + 4)) {
            const StvDTab &d = tabs[x.arg];
            const StvTerm *tm = (const StvTerm *)&b[at + d.term_off];
            for (int i = 0; i < d.nterm; ++i) {
                dep |= 1ull << tm[i].b;
                if (tm[i].a <= -2) dep |= 1ull << (-2 - tm[i].a);
            }
        }
        return dep;
    };
    std::vector<StvTcStep> st;
    int nop = 0;
    uint64_t dep_all = 0;
    auto build = [&](bool allow_bvar) {
    st.clear();
    nop = 0;
    dep_all = 0;
    for (size_t gi = 0; gi < grecs.size(); ++gi) {
        const StvGroup &G = grecs[gi];
        const StvSub *sp = (const StvSub *)&b[at + G.sub_off];
        const size_t g0 = st.size();
        bvraw = (allow_bvar && G.nvb >= 8 && hd.S == 12) ? G.vbit[7][0] : 0;
        int k = 0;
        while (k < G.nsub) {
            bool f = foldable(sp[k]);
            int e = k;
            double c = 0;
            uint64_t dep = 0;
            bool bv = false;
            while (e < G.nsub && foldable(sp[e]) == f) {
                c += cost(sp[e]);
                dep |= depends(sp[e]);
                bv |= fold_kind(sp[e]) == 2;
                ++e;
            }
            if (f && c < tc_min) f = false;
            if (!f && st.size() > g0 && st.back().kind == 0) {
                st.back().n = (int16_t)(st.back().n + (e - k));
            } else {
                StvTcStep s;
                std::memset(&s, 0, sizeof(s));
                s.kind = f ? 1 : 0;
                s.first = (int16_t)k;
                s.n = (int16_t)(e - k);
                s.group = (int32_t)gi;
                if (f) {
                    s.op = nop;
                    s.bvar = bv ? 1 : 0;
                    nop += bv ? 2 : 1;   // block variants: slots op (block 0) and op + 1 (block 1)
                    s.dep = dep;
                    dep_all |= dep;
                }
                st.push_back(s);
            }
            k = e;
        }
        if (st.size() == g0) {   // no sub-ops (flips only)
            StvTcStep s;
            std::memset(&s, 0, sizeof(s));
            s.group = (int32_t)gi;
            st.push_back(s);
        }
        st.back().last = 1;
    }
    };
    // block variants cost operator slots (2 per step); measured on c2/c4 they pay even where
    // the extra slots push a pass to the single-buffered tile ring
    build(true);
    // the operator slots share the CTA's shared memory with one tile and the phase tables
    // (launch_tc_group_pass): a pass whose block variants do not fit drops them, and runs on
    // the FMA group pass if its operators still do not fit
    auto fits = [&](int slots) {
        return (size_t)STV_TC_SH_BYTES + (size_t)slots * STV_TC_OP_BYTES + 512 +
                   (((size_t)hd.tab_entries * 8 + 127u) & ~(size_t)127) + ((size_t)8 << hd.S) <=
               (size_t)STV_TC_SMEM_CAP;
    };
    if (nop > 0 && nop <= STV_TC_MAX_OPS && !fits(nop)) build(false);
    if (nop > 0 && !fits(nop)) return;   // FMA group pass
    const int nord = __builtin_popcountll(hd.out_mask);
    const size_t need = st.size() * sizeof(StvTcStep) + 16;
    if (nop == 0 || nop > STV_TC_MAX_OPS || st.size() > STV_TC_MAX_STEPS || nord > 48 ||
        grecs.size() > STV_TC_MAX_GROUPS ||
        b.size() - at + need > (size_t)STV_REC_PARAM_BYTES)
        return;   // FMA group pass
    // tile order: ordinal bits the operators depend on vary slowest within a CTA's range
    std::vector<int> lo, hi;
    for (int i = 0; i < nord; ++i) ((dep_all >> nth_set_bit(hd.out_mask, i)) & 1 ? hi : lo).push_back(i);
    int q = 0;
    for (int i : lo) hd.tperm[q++] = (uint8_t)i;
    for (int i : hi) hd.tperm[q++] = (uint8_t)i;
    align(b, 16);
    hd.tc_off = (uint32_t)(b.size() - at);
    hd.ntc = (int32_t)st.size();
    hd.ntcop = nop;
    hd.swz_tma = g_swz_tma ? 1 : 0;
    put(b, st.data(), st.size() * sizeof(StvTcStep));
}

Encoded encode(const Plan &p, int n_local, bool c128, uint64_t rank_bits) {
    Encoded e;
    std::vector<uint8_t> &b = e.blob;
    const size_t esz = c128 ? 16 : 8;
    auto encode_pass = [&](const PPass &ps) {
        align(b, 256);
        const size_t at = b.size();
        e.pass_off.push_back((uint32_t)at);
        StvPass hd;
        std::memset(&hd, 0, sizeof(hd));
        std::vector<uint8_t> tail;                   // global-only part of the record
        hd.kind = ps.kind;
        hd.n_local = n_local;
        b.resize(at + sizeof(StvPass));
        int loc[64];
        for (int i = 0; i < 64; ++i) loc[i] = -1;
        if (ps.kind == PASS_TILE) {
            std::vector<int> sb = bits_of(ps.S);
            int L = 0;
            while (L < (int)sb.size() && sb[L] == L) ++L;
            hd.S = (int)sb.size();
            hd.L = L;
            hd.h = hd.S - L;
            for (int r = 0; r < hd.h; ++r) hd.hpos[r] = sb[L + r];
            for (int i = 0; i < hd.S; ++i) loc[sb[i]] = i;
            const uint64_t lm = n_local >= 64 ? ~0ull : ((1ull << n_local) - 1);
            hd.out_mask = lm & ~ps.S;
            hd.nops = (int)ps.ops.size();
            align(b, 16);
            hd.ops_off = (uint32_t)(b.size() - at);
            const size_t ops_at = b.size();
            bool grouped = !ps.ops.empty();
            for (auto &o : ps.ops) grouped &= (o.type == OP_GROUP);
            b.resize(ops_at + ps.ops.size() * (grouped ? sizeof(StvGroup) : sizeof(StvOp)));
            std::vector<StvOp> recs(ps.ops.size());
            std::vector<std::vector<StvSub>> subs(ps.ops.size());
            std::vector<std::vector<int>> gpos(ps.ops.size());   // group tile positions (sorted)
            auto put_matrix = [&](const std::vector<cd> &M) -> uint32_t {
                const uint32_t off = (uint32_t)(b.size() - at - hd.mat_off);
                for (const cd &z : M) {
                    if (c128) { double v[2] = {z.real(), z.imag()}; put(b, v, 16); }
                    else { float v[2] = {(float)z.real(), (float)z.imag()}; put(b, v, 8); }
                }
                align(b, 16);
                return off;
            };
            // matrices
            align(b, 16);
            hd.mat_off = (uint32_t)(b.size() - at);
            for (size_t i = 0; i < ps.ops.size(); ++i) {
                const FOp &o = ps.ops[i];
                StvOp &r = recs[i];
                std::memset(&r, 0, sizeof(r));
                r.type = o.type;
                r.c_loc = r.c_phys = -1;
                if (o.type == OP_DENSE) {
                    r.k = (int)o.tg.size();
                    for (int j = 0; j < r.k; ++j) r.tpos[j] = loc[o.tg[j]];
                    r.mat_off = put_matrix(o.M);
                } else if (o.type == OP_CNOT) {
                    r.t_loc = loc[o.t];
                    if (loc[o.c] >= 0) r.c_loc = loc[o.c];
                    else r.c_phys = o.c;
                } else if (o.type == OP_GROUP) {
                    // group positions: its tile bits, padded to 4 with unused tile positions
                    std::vector<int> pos;
                    for (int p : bits_of(o.T)) pos.push_back(loc[p]);
                    for (int q = 0; (int)pos.size() < STV_GROUP_BITS && q < hd.S; ++q)
                        if (std::find(pos.begin(), pos.end(), q) == pos.end()) pos.push_back(q);
                    std::sort(pos.begin(), pos.end());
                    gpos[i] = pos;
                    auto lbit = [&](int phys) {
                        const int tp = loc[phys];
                        return (int)(std::find(pos.begin(), pos.end(), tp) - pos.begin());
                    };
                    for (const FOp &so : o.subs) {
                        StvSub sub;
                        std::memset(&sub, 0, sizeof(sub));
                        if (so.type == OP_DENSE) {
                            const int x = lbit(so.tg[0]);
                            static const int pidx[4][4] = {{-1, 0, 1, 2}, {-1, -1, 3, 4}, {-1, -1, -1, 5}, {-1, -1, -1, -1}};
                            // a real matrix (Hadamard, CNOT/X factors, real rotations) takes half the
                            // multiplies: each complex amplitude is scaled by real entries
                            bool real = so.Mv.empty();
                            for (const cd &z : so.M) real = real && std::abs(z.imag()) <= 1e-15 * std::max(1.0, std::abs(z.real()));
                            if (real) {
                                sub.code = so.tg.size() == 1 ? SUBC_U1R + x : SUBC_U2R + pidx[x][lbit(so.tg[1])];
                                const uint32_t off = (uint32_t)(b.size() - at - hd.mat_off);
                                for (const cd &z : so.M) {
                                    if (c128) { double v = z.real(); put(b, &v, 8); }
                                    else { float v = (float)z.real(); put(b, &v, 4); }
                                }
                                align(b, 16);
                                sub.arg = off;
                            } else if (so.tg.size() == 1) sub.code = SUBC_U1 + x;
                            else sub.code = (so.Mv.empty() ? SUBC_U2 : SUBC_U2V) + pidx[x][lbit(so.tg[1])];
                            if (real) {}
                            else if (so.Mv.empty()) sub.arg = put_matrix(so.M);
                            else {
                                // selectors on local bits become bits of the tile ordinal t (base =
                                // pdep(t, out_mask)); global-bit selectors are fixed for this rank
                                std::vector<int> tsel;                 // tile-ordinal bit per kept selector
                                std::vector<size_t> keep;
                                uint32_t vfix = 0;
                                for (size_t q = 0; q < so.sel.size(); ++q) {
                                    const int p = so.sel[q];
                                    if (p < n_local) {
                                        tsel.push_back(__builtin_popcountll(hd.out_mask & ((1ull << p) - 1)));
                                        keep.push_back(q);
                                    } else if ((rank_bits >> p) & 1) vfix |= 1u << q;
                                }
                                for (size_t v = 0; v < ((size_t)1 << keep.size()); ++v) {
                                    uint32_t full = vfix;
                                    for (size_t q = 0; q < keep.size(); ++q)
                                        if ((v >> q) & 1) full |= 1u << keep[q];
                                    const uint32_t off = put_matrix(so.Mv[full]);
                                    if (v == 0) sub.arg = off;
                                }
                                if (keep.empty()) sub.code = SUBC_U2 + (sub.code - SUBC_U2V);
                                for (size_t q = 0; q < 3; ++q) {
                                    const uint32_t c = q < tsel.size() ? (uint32_t)tsel[q] : 31u;   // 31: always 0
                                    sub.code |= (int32_t)(c << (8 + 5 * q));
                                }
                            }
                        } else if (so.type == OP_CNOT) {
                            int c = -1;
                            // a control on one of the group's 4 positions (a T bit or a padding
                            // position) varies inside the register vector: in-register control
                            if (loc[so.c] >= 0 && std::find(pos.begin(), pos.end(), loc[so.c]) != pos.end())
                                c = lbit(so.c);
                            else if (loc[so.c] >= 0) sub.ctl = 1u << loc[so.c];
                            else sub.ctl = (uint32_t)(so.c + 1) << 16;
                            sub.code = SUBC_CNOT + 4 * (c + 1) + lbit(so.t);
                        } else {
                            sub.code = SUBC_DIAG;
                        }
                        subs[i].push_back(sub);
                    }
                }
            }
            hd.mat_bytes = (uint32_t)(b.size() - at - hd.mat_off);
            // diag records of standalone DIAG ops
            for (size_t i = 0; i < ps.ops.size(); ++i) {
                if (ps.ops[i].type != OP_DIAG) continue;
                align(b, 16);
                recs[i].diag_off = (uint32_t)(b.size() - at);
                size_t rec_at = b.size();
                b.resize(rec_at + sizeof(StvDiag));
                encode_diag(b, rec_at, ps.ops[i].form, loc, hd.S);
            }
            // group records: diag tables (static phases + per-tile terms), sub-op arrays
            std::vector<StvDTab> tabs;
            std::vector<StvGroup> grecs(ps.ops.size());
            uint32_t ent = 0;
            for (size_t i = 0; i < ps.ops.size(); ++i) {
                const FOp &o = ps.ops[i];
                if (o.type != OP_GROUP) continue;
                const std::vector<int> &pos = gpos[i];
                std::vector<StvSub> out;
                size_t di = 0;
                for (size_t k = 0; k < o.subs.size(); ++k) {
                    const FOp &so = o.subs[k];
                    if (so.type != OP_DIAG) { out.push_back(subs[i][k]); continue; }
                    (void)di;
                    for (const GroupTable &gt : split_group_diag(so.form, pos, loc)) {
                        StvDTab d;
                        std::memset(&d, 0, sizeof(d));
                        d.m = (int)gt.vpos.size();
                        d.half = gt.half >= 0 ? 1 : 0;
                        for (int v = 0; v < d.m; ++v) d.vraw[v] = (uint16_t)(1u << gt.vpos[v]);
                        d.nterm = (int)gt.terms.size();
                        // static phases live in the global-only tail of the record (read per lane
                        // from device memory, never part of the kernel-parameter copy)
                        align(tail, 16);
                        d.stat_off = (uint32_t)tail.size();
                        put(tail, gt.stat.data(), gt.stat.size() * sizeof(uint64_t));
                        align(tail, 16);
                        d.cstat_off = (uint32_t)tail.size();
                        for (uint64_t ph : gt.stat) {
                            const double a = angle_of_turns(ph);
                            if (c128) { double v[2] = {std::cos(a), std::sin(a)}; put(tail, v, 16); }
                            else { float v[2] = {(float)std::cos(a), (float)std::sin(a)}; put(tail, v, 8); }
                        }
                        align(b, 16);
                        d.term_off = (uint32_t)(b.size() - at);
                        put(b, gt.terms.data(), gt.terms.size() * sizeof(StvTerm));
                        d.ent_off = ent;
                        ent += (uint32_t)((d.half ? STV_TAB_STRIDE_H : STV_TAB_STRIDE) << d.m);
                        StvSub sub;
                        std::memset(&sub, 0, sizeof(sub));
                        sub.code = d.half ? SUBC_DIAGH + gt.half : SUBC_DIAG;
                        sub.arg = (uint32_t)tabs.size();
                        tabs.push_back(d);
                        out.push_back(sub);
                    }
                }
                // adjacent 2-qubit sub-ops on complementary pairs run as one sub-op (one dispatch,
                // interleaved FFMA2 chains); they act on disjoint bits, so order is irrelevant
                {
                    std::vector<StvSub> fused;
                    auto pair_of = [](int code) -> int {
                        const int c = code & 0xff;
                        if (c >= SUBC_U2 && c < SUBC_U2 + 6) return c - SUBC_U2;
                        if (c >= SUBC_U2V && c < SUBC_U2V + 6) return c - SUBC_U2V;
                        return -1;
                    };
                    static const int comp[6] = {5, 4, 3, 2, 1, 0};   // 01<->23, 02<->13, 03<->12
                    static const int pairing[6] = {0, 1, 2, 2, 1, 0};
                    for (size_t k = 0; k < out.size(); ++k) {
                        const int pa = pair_of(out[k].code);
                        if (pa >= 0 && k + 1 < out.size() && pair_of(out[k + 1].code) == comp[pa]) {
                            StvSub f;
                            std::memset(&f, 0, sizeof(f));
                            const StvSub &A = pa < comp[pa] ? out[k] : out[k + 1];
                            const StvSub &B = pa < comp[pa] ? out[k + 1] : out[k];
                            auto sel_bits = [](const StvSub &x) -> uint32_t {   // 3 x 5-bit selectors
                                const int c = x.code & 0xff;
                                if (c >= SUBC_U2V) return (uint32_t)x.code >> 8;
                                return 31u | (31u << 5) | (31u << 10);        // plain: never selects
                            };
                            f.code = (int32_t)((SUBC_U2X2 + pairing[pa]) | (sel_bits(A) << 8));
                            f.arg = A.arg;
                            f.ctl = B.arg;
                            f.pad = sel_bits(B);
                            fused.push_back(f);
                            ++k;
                        } else fused.push_back(out[k]);
                    }
                    out = fused;
                }
                // CNOT sub-ops whose control is not a register bit are predicated X flips of a
                // local bit; at the very start / end of the program (moved past ops that do not
                // touch the bit; X flips commute with each other) they cost nothing: the gather /
                // scatter address of local index l becomes that of l xor flips (pass_format.h)
                std::vector<uint32_t> gflips, sflips;
                {
                    auto is_flip = [&](const StvSub &x) {
                        const int c = x.code & 0xff;
                        if (!(c >= SUBC_CNOT && c < SUBC_CNOT + 4)) return false;   // in-register control -1
                        // complex64 pair accesses (16 B) cannot swap the two amplitudes of a pair
                        return c128 || pos[c - SUBC_CNOT] != 0;
                    };
                    auto touches = [&](const StvSub &x, int t) -> bool {  // local bits an op involves
                        const int c = x.code & 0xff;
                        if (c < SUBC_U2) return c - SUBC_U1 == t;
                        if (c < SUBC_CNOT) { const int p = c - SUBC_U2; static const int A[6] = {0,0,0,1,1,2}, Bb[6] = {1,2,3,2,3,3}; return A[p] == t || Bb[p] == t; }
                        if (c < SUBC_DIAG) { const int cc = (c - SUBC_CNOT) / 4 - 1, tt = (c - SUBC_CNOT) % 4; return tt == t || cc == t; }
                        if (c >= SUBC_U1R && c < SUBC_U2R) return c - SUBC_U1R == t;
                        if (c >= SUBC_U2R && c < SUBC_U2R + 6) { const int p = c - SUBC_U2R; static const int A[6] = {0,0,0,1,1,2}, Bb[6] = {1,2,3,2,3,3}; return A[p] == t || Bb[p] == t; }
                        if (c >= SUBC_U2V && c < SUBC_U2V + 6) { const int p = c - SUBC_U2V; static const int A[6] = {0,0,0,1,1,2}, Bb[6] = {1,2,3,2,3,3}; return A[p] == t || Bb[p] == t; }
                        return true;                                      // tables, fused pairs: all bits
                    };
                    auto encode_flip = [&](const StvSub &x) -> uint32_t {
                        const int t = ((x.code & 0xff) - SUBC_CNOT) % 4;
                        const uint32_t dlt = swz_amp(1u << pos[t], c128);
                        if (x.ctl & 0xffffu) return dlt | ((x.ctl & 0xffffu) << 17);
                        return dlt | (1u << 16) | (((x.ctl >> 16) - 1) << 17);
                    };
                    bool moved = true;
                    while (moved && (int)gflips.size() < STV_MAX_FLIPS) {
                        moved = false;
                        for (size_t k = 0; k < out.size(); ++k) {
                            if (!is_flip(out[k])) continue;
                            const int t = ((out[k].code & 0xff) - SUBC_CNOT) % 4;
                            bool ok = true;
                            for (size_t q = 0; q < k && ok; ++q) ok = is_flip(out[q]) || !touches(out[q], t);
                            if (!ok) continue;
                            gflips.push_back(encode_flip(out[k]));
                            out.erase(out.begin() + (long)k);
                            moved = true;
                            break;
                        }
                    }
                    moved = true;
                    while (moved && (int)sflips.size() < STV_MAX_FLIPS) {
                        moved = false;
                        for (size_t k = out.size(); k-- > 0;) {
                            if (!is_flip(out[k])) continue;
                            const int t = ((out[k].code & 0xff) - SUBC_CNOT) % 4;
                            bool ok = true;
                            for (size_t q = k + 1; q < out.size() && ok; ++q) ok = is_flip(out[q]) || !touches(out[q], t);
                            if (!ok) continue;
                            sflips.push_back(encode_flip(out[k]));
                            out.erase(out.begin() + (long)k);
                            moved = true;
                            break;
                        }
                    }
                }
                subs[i] = out;
                StvGroup &g = grecs[i];
                std::memset(&g, 0, sizeof(g));
                for (int j = 0; j < 4; ++j) g.tpos[j] = pos[j];
                g.nvb = hd.S - STV_GROUP_BITS;
                g.pair16 = (!c128 && pos[0] == 0) ? 1 : 0;
                bool v7free = false;
                std::vector<int> vp = vector_bit_order(pos, hd.S, c128);
                if (!c128 && g.nvb >= 8 && hd.S == 12) {
                    // tensor-core block variant (tc_pass.cuh): the in-tile bit outside the group
                    // that its one-V-bit tables and V-bit-controlled CNOTs use most becomes vector
                    // bit 7 (= the TMEM block of a vector), so those sub-ops are tile-uniform within
                    // a block and fold into per-block operators; lane bits (order head) stay
                    std::map<int, int> cnt;
                    for (const StvSub &x : out) {
                        const int c = x.code & 0xff;
                        if ((c == SUBC_DIAG || (c >= SUBC_DIAGH && c < SUBC_DIAGH + 4)) && tabs[x.arg].m == 1)
                            cnt[__builtin_ctz(tabs[x.arg].vraw[0])]++;
                        if (c >= SUBC_CNOT && c < SUBC_DIAG && (x.ctl & 0xffffu) && !((x.ctl & 0xffffu) & ((x.ctl & 0xffffu) - 1)))
                            cnt[__builtin_ctz(x.ctl & 0xffffu)]++;
                    }
                    int best = -1, bc = 0;
                    for (auto &kv : cnt)
                        if (kv.second > bc) { best = kv.first; bc = kv.second; }
                    if (best >= 0) vp = vector_bit_order(pos, hd.S, c128, best);
                    auto it = std::find(vp.begin(), vp.end(), best);
                    // (lane bits of a shared-memory phase: vector bits 0..2 for 16-B accesses, 0..3
                    // for 8-B accesses; STV_V7_STRICT=1: 0..3 for both, the earlier rule)
                    static const bool strict = getenv("STV_V7_STRICT") != nullptr;
                    const int nlane = (g.pair16 && !strict) ? 3 : 4;
                    if (best >= 0 && it != vp.end() && it - vp.begin() >= nlane) std::swap(*it, vp[7]);
                    v7free = best < 0;   // no block variant: vector bit 7 is chosen after the loop
                }
                for (int v = 0; v < g.nvb; ++v) {
                    g.vbit[v][0] = 1u << vp[v];
                    g.vbit[v][1] = swz_amp(1u << vp[v], c128);
                }
                for (int l = 0; l < 16; ++l) {
                    uint32_t off = 0;
                    for (int j = 0; j < 4; ++j)
                        if ((l >> j) & 1) off |= 1u << pos[j];
                    g.sw_off[l] = swz_amp(off, c128);
                }
                {   // per-thread vector bases of the first 8 vector bits (kernel: one load per group)
                    align(tail, 16);
                    g.vtab_off = (uint32_t)tail.size();
                    for (uint32_t t = 0; t < 256; ++t) {
                        uint32_t raw = 0, sw = 0;
                        for (int v = 0; v < std::min(g.nvb, 8); ++v)
                            if ((t >> v) & 1) { raw |= g.vbit[v][0]; sw ^= g.vbit[v][1]; }
                        const uint32_t w = (sw & 0xffffu) | (raw << 16);
                        put(tail, &w, 4);
                    }
                }
                g.pad = v7free ? 1 : 0;   // read by the vector-bit-7 pass below, then cleared
                g.nflip_g = (int)gflips.size();
                g.nflip_s = (int)sflips.size();
                for (size_t q = 0; q < gflips.size(); ++q) g.flip[q] = gflips[q];
                for (size_t q = 0; q < sflips.size(); ++q) g.flip[STV_MAX_FLIPS + q] = sflips[q];
                align(b, 16);
                g.nsub = (int)subs[i].size();
                g.sub_off = (uint32_t)(b.size() - at);
                recs[i].nsub = g.nsub;
                recs[i].sub_off = g.sub_off;
                put(b, subs[i].data(), subs[i].size() * sizeof(StvSub));
            }
            hd.ntab = (int)tabs.size();
            hd.tab_entries = ent;
            align(b, 16);
            hd.tab_off = (uint32_t)(b.size() - at);
            put(b, tabs.data(), tabs.size() * sizeof(StvDTab));
            hd.grouped = grouped ? 1 : 0;
            if (grouped) {
                // a group left with no sub-ops (only predicated X flips) folds into the previous
                // group's scatter: flips commute with nothing in between (they follow all of its
                // ops), and their controls must be fixed for that group's vectors
                for (size_t i = 1; i < grecs.size();) {
                    StvGroup &G2 = grecs[i], &G1 = grecs[i - 1];
                    bool ok = G2.nsub == 0 && G1.nflip_s + G2.nflip_g + G2.nflip_s <= STV_MAX_FLIPS;
                    auto ctl_ok = [&](uint32_t f) {
                        if (f & (1u << 16)) return true;
                        const uint32_t raw = f >> 17;
                        for (int j = 0; j < 4; ++j)
                            if (raw == (1u << G1.tpos[j])) return false;     // varies in G1's vectors
                        return true;
                    };
                    // the flipped position must be one of G1's register bits: a flip of a vector
                    // bit would make G1's thread for vector v scatter into vector v^t's slots
                    // (another thread's, with no barrier between gather and scatter)
                    auto tgt_ok = [&](uint32_t f) {
                        for (int j = 0; j < 4; ++j)
                            if ((f & 0xffffu) == G1.sw_off[1u << j]) return true;
                        return false;
                    };
                    for (int q = 0; q < G2.nflip_g && ok; ++q)
                        ok = ctl_ok(G2.flip[q]) && tgt_ok(G2.flip[q]) && !(G1.pair16 && (G2.flip[q] & 1u));
                    for (int q = 0; q < G2.nflip_s && ok; ++q)
                        ok = ctl_ok(G2.flip[STV_MAX_FLIPS + q]) && tgt_ok(G2.flip[STV_MAX_FLIPS + q]) &&
                             !(G1.pair16 && (G2.flip[STV_MAX_FLIPS + q] & 1u));
                    if (!ok) { ++i; continue; }
                    for (int q = 0; q < G2.nflip_g; ++q) G1.flip[STV_MAX_FLIPS + G1.nflip_s++] = G2.flip[q];
                    for (int q = 0; q < G2.nflip_s; ++q) G1.flip[STV_MAX_FLIPS + G1.nflip_s++] = G2.flip[STV_MAX_FLIPS + q];
                    grecs.erase(grecs.begin() + (long)i);
                }
                // Vector bit 7 of the groups without a block variant: the tile position that the
                // previous group maps to vector bit 7 if it is a V-bit here, else one the next group
                // will share, with the lane bits re-chosen around it (vector_bit_order's `avoid`).  Thread t's half t >> 7 then holds
                // the same amplitudes in both groups, and the tensor-core pass separates them with
                // a per-half barrier instead of a CTA barrier (tc_pass.cuh hsync)
                static const bool v7chain = !getenv("STV_NO_V7CHAIN");
                for (size_t i = 0; i < grecs.size(); ++i) {
                    StvGroup &G = grecs[i];
                    const bool freeb = G.pad != 0;
                    G.pad = 0;
                    if (!freeb || !v7chain || c128 || hd.S != 12 || G.nvb != 8) continue;
                    const std::vector<int> pos(G.tpos, G.tpos + 4);
                    auto in = [](const StvGroup &X, int q) {
                        for (int j = 0; j < 4; ++j)
                            if (X.tpos[j] == q) return true;
                        return false;
                    };
                    int want = -1;
                    if (i) {
                        const int q = __builtin_ctz(grecs[i - 1].vbit[7][0]);
                        if (!in(G, q)) want = q;
                    }
                    if (want < 0 && i + 1 < grecs.size()) {
                        const StvGroup &N = grecs[i + 1];
                        if (!N.pad) {   // fixed: its vector bit 7
                            const int q = __builtin_ctz(N.vbit[7][0]);
                            if (!in(G, q)) want = q;
                        } else {        // free as well: the highest position outside both groups
                            for (int q = hd.S - 1; q >= 0 && want < 0; --q)
                                if (!in(G, q) && !in(N, q)) want = q;
                        }
                    }
                    if (want < 0) continue;
                    std::vector<int> vp = vector_bit_order(pos, hd.S, c128, want);
                    auto it = std::find(vp.begin(), vp.end(), want);
                    // vector bits 0..2 (16-B accesses, pair16) or 0..3 (8-B accesses) are the
                    // conflict-free lane bits of a shared-memory phase
                    if (it == vp.end() || it - vp.begin() < (G.pair16 ? 3 : 4)) continue;
                    std::swap(*it, vp[7]);
                    for (int v = 0; v < 8; ++v) {
                        G.vbit[v][0] = 1u << vp[v];
                        G.vbit[v][1] = swz_amp(1u << vp[v], c128);
                    }
                    for (uint32_t t = 0; t < 256; ++t) {   // its per-thread vector bases
                        uint32_t raw = 0, sw = 0;
                        for (int v = 0; v < 8; ++v)
                            if ((t >> v) & 1) { raw |= G.vbit[v][0]; sw ^= G.vbit[v][1]; }
                        const uint32_t w = (sw & 0xffffu) | (raw << 16);
                        std::memcpy(&tail[G.vtab_off + 4 * t], &w, 4);
                    }
                }
                hd.nops = (int)grecs.size();
                std::memcpy(&b[ops_at], grecs.data(), grecs.size() * sizeof(StvGroup));
                // tensor-core steps on full 4096-amplitude tiles only: a smaller tile leaves most of
                // the 256 threads (one per 16-amplitude vector) idle, and the CUDA-core pass is
                // faster there (c1, n = 16: 0.38 vs 0.45 ms); STV_TC_SMALL=1 keeps the tensor-core
                // pass for tiles of < 12 bits too (tests)
                static const bool tc_small = getenv("STV_TC_SMALL") && atoi(getenv("STV_TC_SMALL"));
                if (!c128 && !(p.flags & SV_OPT_NO_TC) && (hd.S == 12 || (tc_small && hd.S < 12)))
                    encode_tc_steps(b, at, hd, grecs, tabs);
            }
            else std::memcpy(&b[ops_at], recs.data(), recs.size() * sizeof(StvOp));
            (void)esz;
        } else if (ps.kind == PASS_DIAG) {
            int S = std::min(n_local, 12);
            hd.S = S;
            hd.L = S;
            hd.h = 0;
            for (int i = 0; i < S; ++i) loc[i] = i;
            const uint64_t lm = n_local >= 64 ? ~0ull : ((1ull << n_local) - 1);
            hd.out_mask = lm & ~((1ull << S) - 1);
            align(b, 16);
            hd.diag_off = (uint32_t)(b.size() - at);
            size_t rec_at = b.size();
            b.resize(rec_at + sizeof(StvDiag));
            encode_diag(b, rec_at, ps.ops[0].form, loc, S);
        } else if (ps.kind == PASS_CNOT) {
            hd.cnot_c = ps.ops[0].c;
            hd.cnot_t = ps.ops[0].t;
        }
        align(b, 16);
        hd.param_bytes = (uint32_t)(b.size() - at);
        if (!tail.empty()) {                         // global-only tail: patch the offsets into it
            const uint32_t base = (uint32_t)(b.size() - at);
            for (int t = 0; t < hd.ntab; ++t) {
                StvDTab *d = (StvDTab *)&b[at + hd.tab_off + (size_t)t * sizeof(StvDTab)];
                d->stat_off += base;
                d->cstat_off += base;
            }
            if (hd.grouped)
                for (int i = 0; i < hd.nops; ++i) {
                    StvGroup *g = (StvGroup *)&b[at + hd.ops_off + (size_t)i * sizeof(StvGroup)];
                    g->vtab_off += base;
                }
            put(b, tail.data(), tail.size());
            align(b, 16);
        }
        hd.rec_bytes = (uint32_t)(b.size() - at);
        std::memcpy(&b[at], &hd, sizeof(hd));
    };
    for (const PPass &ps : p.passes) {
        // with SV_OPT_TMA, tensor-core candidates are encoded for TMA staging (SWIZZLE_128B tile
        // layout); a pass that ends up without operator steps is re-encoded for the CUDA-core pass
        const bool tma = !c128 && ps.kind == PASS_TILE && __builtin_popcountll(ps.S) <= 12 &&
                         (p.flags & SV_OPT_TMA) && !(p.flags & SV_OPT_NO_TC);
        const size_t mark = b.size();
        g_swz_tma = tma;
        encode_pass(ps);
        if (tma && ((const StvPass *)&b[e.pass_off.back()])->ntc == 0) {
            b.resize(mark);
            e.pass_off.pop_back();
            g_swz_tma = false;
            encode_pass(ps);
        }
        g_swz_tma = false;
    }
    align(b, 256);
    return e;
}

// ---------------------------------------------------------------------------
// JSON (for the CPU plan-interpreter tests)
// ---------------------------------------------------------------------------
static std::string ops_json(const std::vector<FOp> &ops) {
    std::ostringstream o;
    o.precision(17);
    o << "[";
    for (size_t j = 0; j < ops.size(); ++j) {
        const FOp &f = ops[j];
        if (j) o << ",";
        o << "{\"type\":" << f.type;
        if (f.type == OP_DENSE) {
            o << ",\"tg\":[";
            for (size_t t = 0; t < f.tg.size(); ++t) o << (t ? "," : "") << f.tg[t];
            o << "],\"re\":[";
            for (size_t t = 0; t < f.M.size(); ++t) o << (t ? "," : "") << f.M[t].real();
            o << "],\"im\":[";
            for (size_t t = 0; t < f.M.size(); ++t) o << (t ? "," : "") << f.M[t].imag();
            o << "]";
            if (!f.Mv.empty()) {
                o << ",\"sel\":[";
                for (size_t t = 0; t < f.sel.size(); ++t) o << (t ? "," : "") << f.sel[t];
                o << "],\"vre\":[";
                for (size_t v = 0; v < f.Mv.size(); ++v) {
                    o << (v ? "," : "") << "[";
                    for (size_t t = 0; t < f.Mv[v].size(); ++t) o << (t ? "," : "") << f.Mv[v][t].real();
                    o << "]";
                }
                o << "],\"vim\":[";
                for (size_t v = 0; v < f.Mv.size(); ++v) {
                    o << (v ? "," : "") << "[";
                    for (size_t t = 0; t < f.Mv[v].size(); ++t) o << (t ? "," : "") << f.Mv[v][t].imag();
                    o << "]";
                }
                o << "]";
            }
        } else if (f.type == OP_DIAG) {
            o << ",\"cst\":\"" << f.form.cst << "\",\"lin\":[";
            bool c = false;
            for (auto &kv : f.form.lin) { o << (c ? "," : "") << "[" << kv.first << ",\"" << kv.second << "\"]"; c = true; }
            o << "],\"quad\":[";
            c = false;
            for (auto &kv : f.form.quad) {
                o << (c ? "," : "") << "[" << kv.first.first << "," << kv.first.second << ",\"" << kv.second << "\"]";
                c = true;
            }
            o << "]";
        } else if (f.type == OP_GROUP) {
            o << ",\"T\":\"" << f.T << "\",\"subs\":" << ops_json(f.subs);
        } else {
            o << ",\"c\":" << f.c << ",\"t\":" << f.t;
        }
        o << "}";
    }
    o << "]";
    return o.str();
}

std::string plan_to_json(const Plan &p) {
    std::ostringstream o;
    o.precision(17);
    o << "{\"n\":" << p.n << ",\"n_global\":" << p.n_global << ",\"alg_bytes\":" << p.alg_bytes << ",\"passes\":[";
    for (size_t i = 0; i < p.passes.size(); ++i) {
        const PPass &ps = p.passes[i];
        if (i) o << ",";
        o << "{\"kind\":" << ps.kind << ",\"S\":" << ps.S << ",\"gates\":[";
        for (size_t j = 0; j < ps.gates.size(); ++j) o << (j ? "," : "") << ps.gates[j];
        o << "],\"swaps\":[";
        for (size_t j = 0; j < ps.swaps.size(); ++j)
            o << (j ? "," : "") << "[" << ps.swaps[j].first << "," << ps.swaps[j].second << "]";
        o << "],\"ops\":" << ops_json(ps.ops) << "}";
    }
    o << "],\"perm\":[";
    for (int q = 0; q < p.n; ++q) o << (q ? "," : "") << p.frame_out.perm[q];
    o << "],\"xmask\":\"" << p.frame_out.xmask << "\"}";
    return o.str();
}


// Estimated cost of an encoded plan in units of one gate-group round on the resident tile
// (measured on one B200, c2/c3/c4 low-bits sweep): every group, operator
// (M) step and register (E) step costs about the same (~0.8 ms per 2^30 amplitudes); a
// pass adds ~0.3 of that on top (its copy overlaps the compute).
static double encoded_cost(const Encoded &e) {
    double c = 0;
    for (uint32_t off : e.pass_off) {
        const StvPass *P = (const StvPass *)&e.blob[off];
        c += 0.3 + (P->grouped ? P->nops : 1) + P->ntc;
    }
    return c;
}

Plan plan_auto(int n, int n_global, int amp_bytes, const std::vector<PGate> &pg, const PlanOptions &opt,
               int *sigma) {
    static const bool off = getenv("STV_NO_AUTO_LOW") && atoi(getenv("STV_NO_AUTO_LOW"));
    const int nl = n - n_global;
    const bool tc = amp_bytes == 8 && !(opt.flags & (SV_OPT_NO_TC | SV_OPT_NO_GROUPS | SV_OPT_ONE_GATE));
    if (off || !opt.low_auto || !tc || opt.tile_bits != 12 || nl < 20) return build_plan(n, n_global, amp_bytes, pg, opt, sigma);
    int best_sigma[64];
    Plan best;
    double best_cost = 0;
    for (int L : {4, 5}) {
        PlanOptions o = opt;
        o.low_bits = L;
        int sg[64];
        std::memcpy(sg, sigma, sizeof(sg));
        Plan p = build_plan(n, n_global, amp_bytes, pg, o, sg);
        const double c = encoded_cost(encode(p, nl, false, 0));
        if (L == 4 || c < best_cost) {
            best = std::move(p);
            best_cost = c;
            std::memcpy(best_sigma, sg, sizeof(best_sigma));
        }
    }
    std::memcpy(sigma, best_sigma, sizeof(best_sigma));
    return best;
}

}  // namespace stv
