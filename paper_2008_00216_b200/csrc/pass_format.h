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

#define STV_GROUP_BITS 4
#define STV_MAX_TABLES 32
#define STV_MAX_VBITS 3          // in-tile bits outside the group a full diag table may index
#define STV_MAX_VBITS_H 6        // ... a half diag table may index
#define STV_MAX_FLIPS 8          // predicated X flips per group folded into gather / scatter addresses

#define STV_MAX_TILE_BITS 14
#define STV_MAX_K 4
#define STV_THREADS 256
#define STV_REC_PARAM_BYTES 24576   // group-pass record = __grid_constant__ kernel parameter
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
    uint32_t tab_off;          // byte offset of StvDTab[ntab]
    int32_t grouped;           // 1: every op is a gate group (StvGroup[nops] at ops_off), k_group_pass
    uint32_t tab_entries;      // total table entries (amplitudes) in shared memory
    uint32_t param_bytes;      // leading bytes of the record passed as the group-pass kernel
                               // parameter (the rest -- static table phases -- is read from
                               // device memory only)
    // tensor-core group pass (tc_pass.cuh; complex64, S <= 12): ntc > 0 selects it
    uint32_t tc_off;           // byte offset of StvTcStep[ntc] (kernel-parameter part)
    int32_t ntc;               // steps over all groups, in group order
    int32_t ntcop;             // operator slots (M steps), <= STV_TC_MAX_OPS
    int32_t swz_tma;           // 1: tile layout = TMA SWIZZLE_128B (chunk c at c ^ ((c >> 3) & 7)), tiles
                               // staged with cp.async.bulk.tensor; 0: the kSwzH pattern below
    uint8_t tperm[48];         // tile ordinal bit of permuted-ordinal bit i (dep bits on top)
};

// Tensor-core pass step: a group's sub-op program [first, first + n) either runs
// on the register vectors (kind 0, "E") or is multiplied into one 16 x 16 complex
// operator applied with tcgen05.mma (kind 1, "M"; slot `op`, rebuilt when the
// tile base bits `dep` change).  `last` ends the group's steps.
#define STV_TC_MAX_OPS 12
#define STV_TC_MAX_STEPS 64
#define STV_TC_MAX_GROUPS 16
// shared memory of the tensor-core pass (tc_pass.cuh): TcShared region | tile ring (1 or 2
// tiles) | operator slots | 512 B of scalars | phase tables; 113 KB per CTA keeps 2 CTAs per SM
#define STV_TC_SH_BYTES 2048
#define STV_TC_OP_BYTES 8192
#define STV_TC_SMEM_CAP (113 * 1024)
struct alignas(16) StvTcStep {
    int16_t kind, last, first, n;
    int32_t op, group;
    uint64_t dep;
    int32_t bvar;              // M: 1 = per-block operator variants (slot op: block 0, op + 1: block 1;
                               // the block is vector bit 7, the step's sub-ops depend on it)
    int32_t pad;
};

// ---------------------------------------------------------------------------
// Gate-group passes (k_group_pass).  A group owns 4 tile positions tpos[0..3]
// (local index bit j <-> tile position tpos[j]); every thread gathers the 16
// amplitudes of one vector (fixed values of the other S-4 "vector" bits) into
// registers, runs the sub-op program and scatters them back.
//
// Shared-memory tile layout (bank-conflict-free gathers): the tile is stored
// in 16-B chunks (2 complex64 / 1 complex128 amplitudes); chunk c lives in slot
//     swz(c) = c ^ H(c >> 3),   H(x) = XOR_j x_j * kSwzH[j]  (3-bit values)
// which is linear over GF(2).  A warp phase of 8 lanes (LDS.128) is
// conflict-free iff its 3 varying chunk bits have independent bank vectors
// (chunk bits 0..2: 1, 2, 4; bit 3+j: kSwzH[j]); the encoder orders every
// group's vector bits so that lane bits 0..2 (0..3 for 8-B accesses) meet that.
// ---------------------------------------------------------------------------
#define STV_SWZ_NH 11
#ifdef __cplusplus
static constexpr uint32_t kSwzH[STV_SWZ_NH] = {3, 5, 6, 7, 1, 2, 4, 3, 5, 6, 7};
static constexpr uint32_t swz_mask(int bit) {
    uint32_t m = 0;
    for (int j = 0; j < STV_SWZ_NH; ++j)
        if ((kSwzH[j] >> bit) & 1) m |= 1u << j;
    return m;
}
static constexpr uint32_t kSwzM0 = swz_mask(0), kSwzM1 = swz_mask(1), kSwzM2 = swz_mask(2);
#endif

// sub-op dispatch codes (low 8 bits of StvSub.code)
#define SUBC_U1 0                // + a (0..3)
#define SUBC_U2 4                // + pair index of (a<b): 01 02 03 12 13 23 -> 0..5
#define SUBC_CNOT 10             // + 4 * (c + 1) + t, c = in-register control or -1
#define SUBC_DIAG 30
#define SUBC_U2V 31              // + pair index: U2 with per-tile variants (selectors in code bits 8..22)
#define SUBC_DIAGH 37            // + j: half-table diagonal on local bit j (arg = table index)
#define SUBC_U2X2 41             // + pairing ({01,23}, {02,13}, {03,12}): two U2 on complementary pairs;
                                 // arg/code bits 8..22 = first (lower pair) matrix / selectors,
                                 // ctl/pad = second matrix / selectors (31 = unused selector)
#define SUBC_U1R 44              // + a: U1 with a real matrix (stored as 4 reals)
#define SUBC_U2R 48              // + pair index: U2 with a real matrix (stored as 16 reals)
#define SUBC_N 54

struct alignas(16) StvSub {
    int32_t code;              // bits 0..7: SUBC_*; U2V: bits 8+5i (i < 3) = selector i, a bit index of the
                               // tile ordinal t (base = pdep(t, out_mask)), 31 = unused (always 0); variant
                               // v (matrices consecutive from arg) has bit i = selector i of this tile --
                               // uniform per CTA, so matrix loads stay uniform (LDCU)
    uint32_t arg;              // U1/U2/U2V: matrix byte offset in the pass matrix area; DIAG: table index
    uint32_t ctl;              // CNOT: bits 0..15 raw tile offset of a control on a vector bit (0 = none);
                               //       bits 16..23 physical control bit + 1 outside the tile (0 = none)
    uint32_t pad;
};

struct alignas(16) StvGroup {
    int32_t nsub;
    uint32_t sub_off;          // byte offset of StvSub[nsub] from the pass record
    int32_t nvb;               // number of vector bits (S - 4)
    int32_t pair16;            // complex64 with tpos[0] == 0: amplitudes l, l|1 share a 16-B chunk
    int32_t tpos[4];
    uint32_t sw_off[16];       // swizzled tile offset (amplitudes) of local index l
    uint32_t vbit[STV_MAX_TILE_BITS - 4][2];   // vector bit b: {raw tile offset 1 << position, swizzled offset}
    uint32_t vtab_off;         // byte offset (pass record, global-only tail) of uint32 vtab[256]:
                               // thread t's first vector, (swizzled base) | (raw base << 16)
    int32_t nflip_g, nflip_s;  // predicated X flips folded into the gather / scatter addresses
    int32_t pad;
    uint32_t flip[2 * STV_MAX_FLIPS];   // [0, nflip_g) gather, [STV_MAX_FLIPS, +nflip_s) scatter:
                                        // bits 0..15 swizzled offset of the flipped tile position,
                                        // bit 16 control outside the tile, bits 17..31 the raw tile
                                        // offset of the (vector-bit) control or its physical bit
};

// Per-tile phase table of one group DIAG sub-op, over index e = l | (r << 4):
// l = the group's local bits, r = its m V-bits (in-tile bits outside the group).
//   phase(e) = stat[e] + sum of the per-tile terms active for this tile
// Per-tile term {a, b, ang}: a >= 0: index bit a of e times bit b of the
// tile's full base; a == -1: bit b of the base; a <= -2: bits (-2 - a) and b.
// Entries live in shared memory at ent_off + r * STV_TAB_STRIDE + l (rows padded against
// bank conflicts between lanes with different r).
struct alignas(16) StvDTab {
    uint32_t stat_off;         // byte offset (pass record) of uint64 stat[(half ? 8 : 16) << m]
    uint32_t cstat_off;        // byte offset of the same static phases as unit complex numbers
                               // (state precision, rounded once from fp64): entry = cstat[e] x
                               // F_low[low index bits] x F_high[V-bit index] built per tile
    uint32_t term_off;         // byte offset of StvTerm[nterm]
    int32_t nterm;
    int32_t m;
    uint32_t ent_off;          // first entry in the shared-memory table area
    int32_t half;              // 0: full table over l (16) x r; 1: half table (below)
    uint16_t vraw[STV_MAX_VBITS_H];   // raw tile offsets of the V-bits (0 for unused)
};
// Half table (code SUBC_DIAGH + j): every term of the diagonal contains local bit j,
// so amplitudes with l_j = 0 are unchanged; the table is over (the 3 other local
// bits in ascending order) x r, rows of 8 entries at stride STV_TAB_STRIDE_H, and
// its per-tile terms are all constants (a == -1 or <= -2).  QFT-like diagonals
// (one target coupled to many qubits) take m <= STV_MAX_VBITS_H V-bits this way.
#define STV_TAB_STRIDE_H 9
#define STV_TAB_STRIDE 17        // entries per table row: 16 + 1 pad (rows of different lanes hit different banks)
