// plan.h -- host-side gate IR, relabel frame and fusion planner.
//
// Pipeline (each step cites the paper passage it generalises):
//   a1  classify gates: DIAG (phase per basis state), PERM (X, CNOT, SWAP),
//       MONO (perm x phases, e.g. fSim(pi/2, phi) = SWAP . diag), DENSE
//       ("diagonal gates act on individual amplitudes",
//        L544-545 P=T^2, Z=T^4, L552 CNOT).
//   a2  relabel frame: SWAP and the SWAP factor of MONO gates permute the
//       logical->physical bit map; X toggles an XOR mask (PAPER.md L250-252,
//       L1224-1228 hushed "SWAPs do not materially affect runtime").
//   a3  commutation-aware reordering: the Sec. 4.5 scan
//       with obstructed/unobstructed qubits, generalised to "absorb every
//       later gate that commutes with all skipped gates".
//   a4  fusion: member matrices multiplied in exact order (complex128) into
//       k-qubit dense ops (Eq. 2 coalescing; L661-669 the
//       simulation plan); diagonal gates aggregated into one phase form per
//       cluster as uint64 fixed-point turns.
#pragma once
#include <complex>
#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "pass_format.h"
#include "../../include/sv.h"

namespace stv {

using cd = std::complex<double>;

// Phase function of a cluster of diagonal gates over physical bits, in uint64
// turns (2^64 = one full turn, so R_k = 2^{64-k} and T = 2^61 are exact):
//   phase(j) = cst + sum_p lin[p] b_p(j) + sum_{p<q} quad[(p,q)] b_p(j) b_q(j)  (mod 2^64)
// Every 1- and 2-qubit diagonal unitary has exactly this form (its 4-entry
// table t gives cst=t00, lin=t01-t00 / t10-t00, quad=t11-t10-t01+t00).
// This generalises the paper's T-layer masks (popcount(m & j) octants,
// PAPER.md L503-512) and per-qubit CZ masks.
struct QForm {
    uint64_t cst = 0;
    std::map<int, uint64_t> lin;
    std::map<std::pair<int, int>, uint64_t> quad;
    void add(const QForm &o);
    uint64_t eval(uint64_t j) const;
    uint64_t qubits() const;
    bool trivial() const;
};

enum class GType { DENSE, DIAG, CNOT };

// A gate in the physical frame (after a2).  Qubits are "virtual physical"
// bits v in [0,n): the bit v holds data at actual position sigma[v], where
// sigma changes only at global-qubit remaps.
struct PGate {
    GType type;
    int nq = 0;
    int q[2] = {-1, -1};      // DENSE: targets in the matrix's order (q[0] = MSB)
    cd U[16];                 // DENSE matrix (2^nq x 2^nq, row-major, q[0] = MSB)
    QForm form;               // DIAG
    int src = -1;             // index in the caller's gate list
    uint64_t qmask() const;   // all qubits touched
    uint64_t dmask() const;   // qubits acted on non-diagonally (DENSE: all; CNOT: target)
};

struct Frame {
    int perm[64];             // logical qubit -> virtual physical bit
    uint64_t xmask = 0;       // over virtual physical bits
    void identity(int n);
};

// A fused op inside one tile pass (before encoding).
struct FOp {
    int type;                 // OP_DENSE / OP_DIAG / OP_CNOT
    std::vector<int> tg;      // DENSE: ascending actual-physical target bits
    std::vector<cd> M;        // DENSE: 2^k x 2^k, local index LSB-first over tg
    QForm form;               // DIAG (actual-physical bits)
    int c = -1, t = -1;       // CNOT (actual-physical bits)
    uint64_t qmask = 0, dmask = 0;
    uint64_t T = 0;           // GROUP: tile bits held in registers (<= 4, actual physical)
    std::vector<FOp> subs;    // GROUP: sub-ops (DENSE k<=2, DIAG, CNOT) applied in registers
    // DENSE 2-qubit sub-op with per-tile variants: Mv[v] is the matrix for the
    // tile whose physical bits sel[i] (all outside the tile) equal bit i of v
    std::vector<std::vector<cd>> Mv;
    std::vector<int> sel;
};

struct PPass {
    int kind;                 // PASS_TILE / PASS_DIAG / PASS_CNOT / PASS_REMAP
    uint64_t S = 0;           // tile bits (actual physical, all local)
    std::vector<FOp> ops;
    std::vector<std::pair<int, int>> swaps;  // PASS_REMAP: (global bit, local bit)
    std::vector<int> gates;   // caller gate indices absorbed (for tests)
};

struct PlanOptions {
    int kmax = 4;
    int tile_bits = 13;       // c64 default (c128: 12)
    int low_bits = 4;
    int budget = 1000;
    uint32_t flags = 0;
    bool low_auto = true;     // low_bits not given: plan_auto picks it (complex64 tensor-core plans)
};

struct Plan {
    int n = 0, n_global = 0;
    std::vector<PPass> passes;
    Frame frame_out;
    int sigma_out[64];        // virtual -> actual physical bit after the plan
    double alg_bytes = 0;     // algorithmic HBM bytes
    double alg_flops = 0;     // algorithmic FP flops of the fused tile passes
    uint32_t flags = 0;       // SV_OPT_* the plan was built with (encoder choices)
};

// Validation (all-or-nothing).  Returns "" if ok, else the error message.
std::string validate(int n, const sv_gate *g, size_t ng);

// a1+a2: translate to physical gates; updates `fr` in place.
std::vector<PGate> to_physical(int n, const sv_gate *g, size_t ng, Frame &fr, uint32_t flags);

// a3+a4 (+ remaps): build passes.  sigma (virtual->actual) updated in place.
Plan build_plan(int n, int n_global, int amp_bytes, const std::vector<PGate> &pg,
                const PlanOptions &opt, int *sigma);

PlanOptions resolve_options(const sv_options *o, int amp_bytes, int n_local);

// build_plan with the tile's contiguous low run chosen per circuit when the caller left it
// open: complex64 tensor-core plans are built for low_bits 4 and 5 and the one with the
// smaller estimated cost (register rounds + operator steps + passes) is kept.
Plan plan_auto(int n, int n_global, int amp_bytes, const std::vector<PGate> &pg, const PlanOptions &opt,
               int *sigma);

// Encode passes into a device blob for the kernels (pass_format.h).
// rank_bits: value of the global bits (actual positions >= n_local) of this rank.
struct Encoded {
    std::vector<uint8_t> blob;
    std::vector<uint32_t> pass_off;   // byte offset of each pass's PassDesc
};
// rank_bits: this rank's global bit values (physical positions >= n_local); selectors of
// per-tile variant ops on global bits are resolved here.
Encoded encode(const Plan &p, int n_local, bool c128, uint64_t rank_bits = 0);

std::string plan_to_json(const Plan &p);

// Algorithmic floating-point work per amplitude of a pass's ops.
double pass_flops_per_amp(const std::vector<FOp> &ops);

// Exact conversion helpers.
uint64_t turns_of_angle(double rad);   // rad/(2 pi) * 2^64, rounded, mod 2^64
double angle_of_turns(uint64_t t);     // in radians, in [-pi, pi)

}  // namespace stv
