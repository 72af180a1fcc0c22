// pass_format.h -- the device-side plan blob shared by the host encoder
// (plan.cpp) and the CUDA kernels (kernels.cu).  Plain POD, 16-B aligned.
//
// A "tile" of a fused pass is the set of 2^S amplitudes that agree on every
// local physical bit outside the tile-bit set S = [0, L) U {hpos[0..h-1]}.
// Tile-local index i: bits [0, L) are physical bits [0, L); bit L+r is
// physical bit hpos[r].  A tile is 2^h contiguous runs of 2^L amplitudes,
// staged in shared memory by TMA bulk copies.
#pragma once
#include <stdint.h>

#define PASS_TILE 1
#define PASS_DIAG 2
#define PASS_CNOT 3
#define PASS_REMAP 4

#define OP_DENSE 1
#define OP_DIAG 2
#define OP_CNOT 3
#define OP_GROUP 4

// sub-ops of a register-resident gate group (OP_GROUP)
#define SUB_U1 1
#define SUB_U2 2
#define SUB_DIAG 3
#define SUB_CNOT 4
#define STV_GROUP_BITS 4
#define STV_MAX_TABLES 32

#define STV_MAX_TILE_BITS 14
#define STV_MAX_K 4
#define STV_THREADS 256
#define STV_THREADS_LOG 8

struct alignas(16) StvTerm {
    int32_t a, b;
    uint64_t ang;
};

// Diagonal phase form relative to one pass's tile bits (see plan.h QForm):
//   phase(i | base) = cst + sum_{p in out} olin + sum_{out pairs} oquad     (per tile)
//                   + sum_{q in tile} (lin[q] + sum_{cross (q,p), b_p(base)} ang) b_q
//                   + sum_{q<r in tile} A[q][r] b_q b_r
struct alignas(16) StvDiag {
    uint64_t cst;
    uint64_t lin[STV_MAX_TILE_BITS];
    uint64_t A[STV_MAX_TILE_BITS][STV_MAX_TILE_BITS];   // symmetric, zero diagonal
    int32_t n_cross, n_olin, n_oquad, all_quarter;       // all_quarter: every coefficient is a multiple of 1/4 turn
    uint32_t cross_off, olin_off, oquad_off, pad;        // byte offsets from this record
    int32_t cross_start[STV_MAX_TILE_BITS + 2];          // cross terms grouped by tile position a
};

struct alignas(16) StvOp {
    int32_t type;
    int32_t k;                 // DENSE: number of targets
    int32_t tpos[6];           // DENSE: ascending tile-local target positions
    uint32_t mat_off;          // DENSE: byte offset of the 2^k x 2^k matrix in the pass matrix area
    int32_t t_loc;             // CNOT: tile-local target position
    int32_t c_loc;             // CNOT: tile-local control position or -1
    int32_t c_phys;            // CNOT: physical control bit (outside the tile) or -1
    uint32_t diag_off;         // DIAG: byte offset of StvDiag from the PassDesc
    int32_t nsub;              // GROUP: number of sub-ops
    uint32_t sub_off;          // GROUP: byte offset of StvSub[nsub] from the PassDesc
    int32_t pad;
};

// One sub-op of a gate group; local bits index the group's tpos[0..3].
struct alignas(16) StvSub {
    int32_t type;              // SUB_*
    int32_t a, b;              // U1: a; U2: a < b (matrix local index bit0 = a, bit1 = b);
                               // CNOT: a = local control or -1, b = local target
    int32_t c_tile;            // CNOT: tile-local control position outside the group, or -1
    int32_t c_phys;            // CNOT: physical control bit outside the tile, or -1
    uint32_t mat_off;          // U1/U2: byte offset in the pass matrix area
    uint32_t gdiag_off;        // DIAG: byte offset of StvGDiag from the PassDesc
    int32_t tbl;               // DIAG: index of its per-tile phase table
};

// Diagonal sub-op over the group's 4 local bits + bits outside the tile:
//   phase = cst + sum_{olin} + sum_{oquad} + sum_j b_j (w[j] + sum_{cross(j,p)}) + sum_{j<k} A[j][k] b_j b_k
struct alignas(16) StvGDiag {
    uint64_t cst;
    uint64_t w[STV_GROUP_BITS];
    uint64_t A[STV_GROUP_BITS][STV_GROUP_BITS];
    int32_t n_cross, n_olin, n_oquad, n_v;            // n_v = total per-vector terms below
    uint32_t cross_off, olin_off, oquad_off, pad2;    // byte offsets from this record (StvTerm arrays)
    // per-vector terms: in-tile bits outside the group ("V-bits", tile positions)
    int32_t n_vlin, n_vquad, n_vcross, n_vout;        // (q) / (q1, q2) / (local j, q) / (q, outside phys p)
    uint32_t vlin_off, vquad_off, vcross_off, vout_off;
};

struct alignas(16) StvPass {
    int32_t kind;
    int32_t S, L, h;
    int32_t hpos[STV_MAX_TILE_BITS];
    uint64_t out_mask;         // local physical bits outside the tile
    uint64_t rank_bits;        // this rank's global bits (already shifted to >= n_local)
    int32_t n_local, nops;
    uint32_t ops_off;          // byte offset of StvOp[nops] from this record
    uint32_t mat_off;          // byte offset of the matrix area
    uint32_t mat_bytes;
    int32_t cnot_c, cnot_t;    // PASS_CNOT (physical bits)
    uint32_t diag_off;         // PASS_DIAG: StvDiag offset (tile = low S bits)
    uint32_t rec_bytes;        // size of this pass record (multiple of 16)
    int32_t ntab;              // per-tile phase tables of group DIAG sub-ops
    uint32_t tab_off;          // byte offset of uint32 StvGDiag offsets, one per table
    int32_t pad2[3];
};
